cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/pytest10.log; tail -6 gpurun_out/pytest10.log
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -2
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench10.json 2> gpurun_out/bench10.err; cat gpurun_out/bench10.json; tail -2 gpurun_out/bench10.err
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench10_ref.json 2> gpurun_out/bench10_ref.err; cat gpurun_out/bench10_ref.json; tail -2 gpurun_out/bench10_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches10.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python scripts/ncu_launches.py gpurun_out/launches10.csv | head -16
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmm_fast_items" -s 2 -c 1 -o gpurun_out/prof10_spmm python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out/prof10_spmm.ncu-rep
