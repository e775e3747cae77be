cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for a in "" "--cold-host-prepare"; do timeout 900 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline $a > gpurun_out/r3g.json 2> gpurun_out/r3g.err; python -c "import json;d=json.load(open('gpurun_out/r3g.json'));print('$a', round(d['value']/1e9,3), round(d['e2e']['value']/1e9,3), d['e2e_cold'])" || tail -3 gpurun_out/r3g.err; done
