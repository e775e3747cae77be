cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k tcgen05 -x 2>&1 | tail -30 > gpurun_out/pytest2_tc.log
cat gpurun_out/pytest2_tc.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/pytest2.log
tail -15 gpurun_out/pytest2.log
timeout 900 python bench.py --steps 5 --warmup 3 --gemm-mode tf32x3 --no-cpu-baseline > gpurun_out/bench2.json 2> gpurun_out/bench2.err
cat gpurun_out/bench2.json; tail -5 gpurun_out/bench2.err
