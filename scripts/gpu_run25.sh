# Round-1 profile refresh #2 (async SpMM + hub hints + staged uploads): bench line, reference arm, launch
# list, one --set full capture of a whole training step.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r25_bench.json 2> gpurun_out/r25_bench.err; tail -c 900 gpurun_out/r25_bench.json; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r25_ref.json 2> gpurun_out/r25_ref.err; tail -c 200 gpurun_out/r25_ref.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r25_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r25_launches_bench.json 2>&1
python scripts/ncu_launches.py gpurun_out/r25_launches.csv | head -20
timeout 1500 ncu --set full --clock-control none --import-source on --launch-skip 93 --launch-count 31 -o gpurun_out/r25_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r25_full.log 2>&1; tail -2 gpurun_out/r25_full.log
for c in c1 c2 c3; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r25_$c.json 2> gpurun_out/r25_$c.err
  python -c "import json;d=json.load(open('gpurun_out/r25_$c.json'));print('$c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['breakdown_ms_per_step'].items()}, round(d['roofline']['frac'],3), d['e2e']['value'])" || tail -5 gpurun_out/r25_$c.err
done
