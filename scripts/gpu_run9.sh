cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/pytest9.log; tail -6 gpurun_out/pytest9.log
for sm in fast exact; do
timeout 600 python bench.py --steps 5 --warmup 2 --spmm-mode $sm --no-cpu-baseline --no-e2e > gpurun_out/bench9_$sm.json 2> gpurun_out/bench9_$sm.err
python -c "import json;d=json.load(open('gpurun_out/bench9_$sm.json'));print('$sm', round(d['ms_per_step'],2), d['breakdown_ms_per_step'], round(d['roofline']['frac'],3))"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches9.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python scripts/ncu_launches.py gpurun_out/launches9.csv | head -16
