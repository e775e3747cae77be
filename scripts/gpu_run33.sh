cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['ms_per_step'],2), d['breakdown_ms_per_step'])"; done
timeout 300 python bench.py --config c5s --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('c5s', round(d['ms_per_step'],2), d['breakdown_ms_per_step'])"
timeout 1500 ncu --set full --clock-control none -k regex:"gemm_tc|softmax" --launch-skip 27 --launch-count 9 -o gpurun_out/r33_gemm -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r33_gemm.log 2>&1; tail -1 gpurun_out/r33_gemm.log
