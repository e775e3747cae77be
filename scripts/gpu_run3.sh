cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python scripts/tc_accuracy.py > gpurun_out/tc_accuracy.txt 2>&1; cat gpurun_out/tc_accuracy.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/pytest3.log
tail -15 gpurun_out/pytest3.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches3.csv python bench.py --steps 1 --warmup 1 --gemm-mode tf32x3 --no-cpu-baseline --no-e2e > gpurun_out/bench3_ncu.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_exact_rows -s 2 -c 1 -o gpurun_out/prof_spmm python bench.py --steps 1 --warmup 1 --gemm-mode tf32x3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 3 -c 3 -o gpurun_out/prof_gemm python bench.py --steps 1 --warmup 1 --gemm-mode tf32x3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out
