cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/pytest8.log; tail -4 gpurun_out/pytest8.log
timeout 600 python bench.py --steps 5 --warmup 2 --gemm-mode tf32x3 --no-cpu-baseline --no-e2e > gpurun_out/bench8.json 2> gpurun_out/bench8.err
python -c "import json;d=json.load(open('gpurun_out/bench8.json'));print(round(d['ms_per_step'],2), d['breakdown_ms_per_step'], round(d['roofline']['frac'],3))"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches8.csv python bench.py --steps 1 --warmup 1 --gemm-mode tf32x3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python scripts/ncu_launches.py gpurun_out/launches8.csv | head -14
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc|spmm" -s 0 -c 8 -o gpurun_out/prof8 python bench.py --steps 1 --warmup 0 --gemm-mode tf32x3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out/prof8.ncu-rep
