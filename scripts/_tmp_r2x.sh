cd $GRAFT_REPO_ROOT; timeout 600 python scripts/sync_probe.py > gpurun_out/sync.log 2>&1; grep ms/step gpurun_out/sync.log; tail -3 gpurun_out/sync.log
