cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -6
timeout 600 python bench.py > gpurun_out/bench14.json 2> gpurun_out/bench14.err; tail -c 1500 gpurun_out/bench14.json; tail -3 gpurun_out/bench14.err
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-aggregate > gpurun_out/bench14_noagg.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/bench14_noagg.json'));print('noagg', d['ms_per_step'], d['breakdown_ms_per_step'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches14.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench14_ncu.json 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"spmm_fast|gemm_tc2" -c 13 -o gpurun_out/r14_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r14_full.log 2>&1; tail -3 gpurun_out/r14_full.log
ls -la gpurun_out/
