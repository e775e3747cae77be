cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k "tcgen05 and not deterministic" 2>&1 | tail -30 > gpurun_out/pytest4_tc.log; tail -30 gpurun_out/pytest4_tc.log
timeout 300 python scripts/tc_accuracy.py > gpurun_out/tc_accuracy4.txt 2>&1; cat gpurun_out/tc_accuracy4.txt
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/pytest4.log; tail -12 gpurun_out/pytest4.log
timeout 900 python bench.py --steps 5 --warmup 3 --gemm-mode tf32x3 --no-cpu-baseline > gpurun_out/bench4.json 2> gpurun_out/bench4.err; cat gpurun_out/bench4.json; tail -3 gpurun_out/bench4.err
