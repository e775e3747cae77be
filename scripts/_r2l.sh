cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "stream or async_pipeline or spmm_fast or hub_l2 or tuning" > gpurun_out/r2l_tests.log 2>&1; tail -3 gpurun_out/r2l_tests.log
for c in c2 c4 c3; do for st in 0 1; do
timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-cold-e2e --tune spmm_stream=$st > gpurun_out/r2l_$c$st.json 2>gpurun_out/r2l_$c$st.err; python -c "import json,sys;d=json.load(open('gpurun_out/r2l_$c$st.json'));print('$c stream=$st', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['breakdown_ms_per_step'].items()}, round(d['roofline']['frac'],3), d['loss'])" || tail -3 gpurun_out/r2l_$c$st.err
done; done
for st in 0 1; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2l_l_c3_$st.csv python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-cold-e2e --tune spmm_stream=$st > /dev/null 2>&1
python scripts/ncu_launches.py gpurun_out/r2l_l_c3_$st.csv | head -8
done
