cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nproc; free -g | head -2
timeout 600 python scripts/c5_rank_step.py 0 --scale 64 > gpurun_out/r2s_c5_64.json 2> gpurun_out/r2s_c5_64.err; cat gpurun_out/r2s_c5_64.json; tail -3 gpurun_out/r2s_c5_64.err
timeout 2400 python scripts/c5_rank_step.py 0 > gpurun_out/r2s_c5_full.json 2> gpurun_out/r2s_c5_full.err; cat gpurun_out/r2s_c5_full.json; tail -3 gpurun_out/r2s_c5_full.err
