# TN with 32-row stages: GeMM parity + TN trace + C4 bench breakdown.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_properties.py tests/test_gpu_model.py tests/test_gpu_flags.py -q -x -p no:cacheprovider 2>&1 | tail -3
python scripts/gemm_shapes.py --trace tn1 2>&1 | sed -n 20,32p
for i in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['ms_per_step'],2), d['breakdown_ms_per_step'], d['gemm_roofline']['frac'])"; done
