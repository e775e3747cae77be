cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
bash scripts/gpu_run.sh r3d suite bench
grep -E "^FAILED|passed|failed" gpurun_out/r3d_pytest.log | tail -5
BENCH_ARGS="--no-cold-e2e" bash scripts/gpu_run.sh r3d cfg:c2 cfg:c3 cfg:c5s launches ncu_gemm
timeout 1200 python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --no-cold-e2e --cpu-full > gpurun_out/r3d_cpufull.json 2> gpurun_out/r3d_cpufull.err; python -c "import json;d=json.load(open('gpurun_out/r3d_cpufull.json'));print(d.get('cpu_full_reference'))"
