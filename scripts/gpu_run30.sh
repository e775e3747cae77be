cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prepare.py -q -p no:cacheprovider -x 2>&1 | tail -4
timeout 1500 python scripts/prepare_probe.py 2>&1 | tail -8
free -g | head -2
