cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/pytest6.log; tail -8 gpurun_out/pytest6.log
for hr in 2048 4096 16384 100000000; do
  timeout 600 python bench.py --steps 3 --warmup 2 --gemm-mode tf32x3 --no-cpu-baseline --no-e2e --heavy-row $hr > gpurun_out/bench6_hr$hr.json 2> gpurun_out/bench6_hr$hr.err
  python -c "import json;d=json.load(open('gpurun_out/bench6_hr$hr.json'));print($hr, round(d['ms_per_step'],2), d['breakdown_ms_per_step'], round(d['roofline']['frac'],3))"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches6.csv python bench.py --steps 1 --warmup 1 --gemm-mode tf32x3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python scripts/ncu_launches.py gpurun_out/launches6.csv | head -20
