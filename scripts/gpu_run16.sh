cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k tcgen05 -x 2>&1 | tail -15
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -4
for k in 1 2; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --gemm-kernel $k > gpurun_out/bench16_k$k.json 2> gpurun_out/bench16_k$k.err
  python -c "import json;d=json.load(open('gpurun_out/bench16_k$k.json'));print('kernel $k', round(d['ms_per_step'],2), d['breakdown_ms_per_step'])" || tail -5 gpurun_out/bench16_k$k.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc2" -c 8 -o gpurun_out/r16_gemm -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r16_gemm.log 2>&1; tail -2 gpurun_out/r16_gemm.log
