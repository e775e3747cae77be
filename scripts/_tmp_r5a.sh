cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
bash scripts/gpu_run.sh r5a suite bench
grep -E "^FAILED|passed|failed" gpurun_out/r5a_pytest.log | tail -5
