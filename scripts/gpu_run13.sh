cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k tcgen05 -x 2>&1 | tail -15
for k in 1 2; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --gemm-kernel $k > gpurun_out/bench13_k$k.json 2> gpurun_out/bench13_k$k.err
  python -c "import json;d=json.load(open('gpurun_out/bench13_k$k.json'));print('kernel $k', round(d['ms_per_step'],2), d['breakdown_ms_per_step'])" || tail -5 gpurun_out/bench13_k$k.err
done
