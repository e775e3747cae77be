cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "stream or async_pipeline or spmm_fast or hub_l2 or tuning" > gpurun_out/r2k_tests.log 2>&1; tail -3 gpurun_out/r2k_tests.log
for c in c2 c4 c3; do for st in 0 1; do
timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-cold-e2e --tune spmm_stream=$st 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$c stream=$st', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['breakdown_ms_per_step'].items()}, round(d['roofline']['frac'],3), d['loss'])"
done; done
