cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tuning.py tests/test_gpu_kernels.py -q -p no:cacheprovider 2>&1 | tail -5
for slab in 0 8 16 32; do
  timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --spmm-slab $slab > gpurun_out/bench11_s$slab.json 2> gpurun_out/bench11_s$slab.err
  python -c "import json;d=json.load(open('gpurun_out/bench11_s$slab.json'));print('slab $slab', round(d['ms_per_step'],2), d['breakdown_ms_per_step'], round(d['roofline']['frac'],3))" || tail -3 gpurun_out/bench11_s$slab.err
done
