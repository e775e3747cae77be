cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_timeline.py -q -p no:cacheprovider 2>&1 | tail -25
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -6
