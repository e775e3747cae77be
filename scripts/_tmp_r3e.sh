cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "v3_variants or tcgen05" 2>&1 | tail -2
for rep in 1 2; do for t in "gemm3_cluster=2" "gemm3_cluster=1"; do timeout 600 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-cold-e2e --tune $t > gpurun_out/r3e.json 2> gpurun_out/r3e.err; python -c "import json;d=json.load(open('gpurun_out/r3e.json'));print('$t', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['breakdown_ms_per_step'].items()}, d['clocks']['sm_mhz'], d['loss'])" || tail -5 gpurun_out/r3e.err; done; done
MG_TUNE=gemm3_cluster=2 timeout 300 python scripts/gemm_shapes.py --trace nn1 > gpurun_out/r3e_trace.txt 2>&1
