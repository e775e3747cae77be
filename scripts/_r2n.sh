cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "stream" > gpurun_out/r2n_tests.log 2>&1; tail -2 gpurun_out/r2n_tests.log
for P in 1 2 4 8; do
timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/r2n_p$P.csv python scripts/p_stage_probe.py $P > gpurun_out/r2n_p$P.log 2>&1; tail -1 gpurun_out/r2n_p$P.log
python scripts/p_stage_probe.py --summarise gpurun_out/r2n_p$P.csv $P > gpurun_out/r2n_p$P.json; python -c "import json;d=json.load(open('gpurun_out/r2n_p$P.json'));print($P, {k: round(v,3) for k,v in d.items() if isinstance(v,float)})"
done
