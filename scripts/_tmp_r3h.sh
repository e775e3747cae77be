cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tuning.py tests/test_gpu_model.py -q -p no:cacheprovider 2>&1 | tail -2
REPS=3 timeout 600 python scripts/e2e_probe.py c4 > gpurun_out/r3h_e2e.log 2>&1; grep -E "lists|tiles |create" gpurun_out/r3h_e2e.log | tail -8
