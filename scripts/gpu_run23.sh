cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in c1 c2 c3; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r23_$c.json 2> gpurun_out/r23_$c.err
  python -c "import json;d=json.load(open('gpurun_out/r23_$c.json'));print('$c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['breakdown_ms_per_step'].items()}, round(d['roofline']['frac'],3), d['e2e']['value'])" || tail -5 gpurun_out/r23_$c.err
done
