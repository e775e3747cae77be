cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python scripts/tc_accuracy.py > gpurun_out/tc_accuracy5.txt 2>&1; cat gpurun_out/tc_accuracy5.txt
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/pytest5.log; tail -12 gpurun_out/pytest5.log
timeout 900 python bench.py --steps 10 --warmup 3 --gemm-mode tf32x3 --no-cpu-baseline > gpurun_out/bench5.json 2> gpurun_out/bench5.err; cat gpurun_out/bench5.json; tail -3 gpurun_out/bench5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches5.csv python bench.py --steps 1 --warmup 1 --gemm-mode tf32x3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 4 -o gpurun_out/prof5_gemm python bench.py --steps 1 --warmup 1 --gemm-mode tf32x3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_exact_heavy -s 1 -c 1 -o gpurun_out/prof5_heavy python bench.py --steps 1 --warmup 1 --gemm-mode tf32x3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls gpurun_out
