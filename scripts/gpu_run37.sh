# Checkpoint: whole GPU suite, smoke(), default bench line.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r37_pytest.log 2>&1; tail -3 gpurun_out/r37_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/r37_bench.json 2> gpurun_out/r37_bench.err; python -c "import json;d=json.load(open('gpurun_out/r37_bench.json'));print(round(d['ms_per_step'],2), d['breakdown_ms_per_step'], d['e2e']['value'], d['clocks'])" || tail -5 gpurun_out/r37_bench.err
