cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -x 2>&1 | tail -8
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for k in 1 2; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --gemm-kernel $k > gpurun_out/bench17_k$k.json 2> gpurun_out/bench17_k$k.err
  python -c "import json;d=json.load(open('gpurun_out/bench17_k$k.json'));print('kernel $k', round(d['ms_per_step'],2), d['breakdown_ms_per_step'])" || tail -5 gpurun_out/bench17_k$k.err
done
for s in 0 16 32; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --spmm-slab $s > gpurun_out/bench17_s$s.json 2> gpurun_out/bench17_s$s.err
  python -c "import json;d=json.load(open('gpurun_out/bench17_s$s.json'));print('slab $s', round(d['ms_per_step'],2), d['breakdown_ms_per_step'])" || tail -5 gpurun_out/bench17_s$s.err
done
