cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "stream or spmm_fast or fast_modes or hub" > gpurun_out/r2o_tests.log 2>&1; tail -2 gpurun_out/r2o_tests.log
for P in 1 2 4 8; do timeout 600 python scripts/p_stage_probe.py $P 5 2>&1 | tail -1; done
for P in 8; do MG_TUNE=spmm_stream=1 timeout 600 python scripts/p_stage_probe.py $P 5 2>&1 | tail -1; done
for c in c2 c4; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-cold-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['breakdown_ms_per_step'].items()}, round(d['roofline']['frac'],3), d['loss'])"; done
