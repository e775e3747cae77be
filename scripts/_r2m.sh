cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "stream or async_pipeline or spmm_fast or hub_l2 or tuning or fast_modes" > gpurun_out/r2m_tests.log 2>&1; tail -2 gpurun_out/r2m_tests.log
for c in c2 c3 c4; do for ad in 0 1; do for st in 0 1; do
timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-cold-e2e --tune spmm_stream=$st --tune adaptive_cuts=$ad > gpurun_out/r2m_$c$ad$st.json 2>gpurun_out/r2m_$c$ad$st.err; python -c "import json,sys;d=json.load(open('gpurun_out/r2m_$c$ad$st.json'));print('$c adaptive=$ad stream=$st', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['breakdown_ms_per_step'].items()}, round(d['roofline']['frac'],3), d['loss'])" || tail -3 gpurun_out/r2m_$c$ad$st.err
done; done; done
