cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do
for t in "gemm_f16=1" "gemm_f16=0" "gemm_f16=1 --tune gemm_f16_min_k=0"; do timeout 600 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-cold-e2e --tune $t > gpurun_out/r2w.json 2> gpurun_out/r2w.err; python -c "import json;d=json.load(open('gpurun_out/r2w.json'));print('$t', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['breakdown_ms_per_step'].items()}, d['clocks']['sm_mhz'])" || tail -5 gpurun_out/r2w.err; done; done
MG_TUNE=gemm_f16=1 timeout 300 python scripts/gemm_shapes.py --trace nn0 > gpurun_out/r2w_trace_nn0.txt 2>&1
