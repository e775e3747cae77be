cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tuning.py -q -p no:cacheprovider -k "stage_fold or solo" > gpurun_out/r2t_t.log 2>&1; tail -4 gpurun_out/r2t_t.log
for f in 0 2 4 7; do MG_TUNE=stage_fold=$f timeout 900 python scripts/p_stage_probe.py 8 5 2>&1 | tail -1; done
timeout 2400 python scripts/c5_rank_step.py 0 > gpurun_out/r2t_c5_full.json 2> gpurun_out/r2t_c5_full.err; cat gpurun_out/r2t_c5_full.json
