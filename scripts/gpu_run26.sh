cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_tuning.py -q -p no:cacheprovider -x -k "async or hub" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -3
for c in c4 c3 c2; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r26_$c.json 2> gpurun_out/r26_$c.err
  python -c "import json;d=json.load(open('gpurun_out/r26_$c.json'));print('$c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['breakdown_ms_per_step'].items()}, round(d['roofline']['frac'],3))" || tail -5 gpurun_out/r26_$c.err
done
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --spmm-async 0 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('c4 regs', round(d['ms_per_step'],2), d['breakdown_ms_per_step'])"
