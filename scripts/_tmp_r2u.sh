cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
REPS=3 timeout 600 python scripts/e2e_probe.py c4 > gpurun_out/r2u_e2e.log 2>&1; grep -v "^\[tc" gpurun_out/r2u_e2e.log | tail -60
