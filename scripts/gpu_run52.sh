# Round-1 profile refresh #10 (final state of round 1): bench line (+ e2e, cpu baseline), reference arm, launch list,
# ncu --set full of one step's SpMM and GeMM kernels, the other configs' bench lines, GPU suite + smoke.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r52_pytest.log 2>&1; tail -1 gpurun_out/r52_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r52_bench.json 2> gpurun_out/r52_bench.err; tail -c 300 gpurun_out/r52_bench.json; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r52_ref.json 2> gpurun_out/r52_ref.err; tail -c 200 gpurun_out/r52_ref.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r52_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r52_launches_bench.json 2>&1
python scripts/ncu_launches.py gpurun_out/r52_launches.csv > gpurun_out/r52_launches.txt; head -14 gpurun_out/r52_launches.txt
timeout 1500 ncu --set full --clock-control none -k regex:"spmm_fast" --launch-skip 30 --launch-count 10 -o gpurun_out/r52_spmm -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r52_spmm.log 2>&1; tail -1 gpurun_out/r52_spmm.log
timeout 1500 ncu --set full --clock-control none -k regex:"gemm_tc|softmax" --launch-skip 27 --launch-count 9 -o gpurun_out/r52_gemm -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r52_gemm.log 2>&1; tail -1 gpurun_out/r52_gemm.log
python scripts/ncu_summary.py gpurun_out/r52_spmm.ncu-rep > gpurun_out/r52_ncu_spmm.txt 2>&1; python scripts/ncu_summary.py gpurun_out/r52_gemm.ncu-rep > gpurun_out/r52_ncu_gemm.txt 2>&1
rm -f gpurun_out/*.ncu-rep
for c in c1 c2 c3 c5s; do
  timeout 1200 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r52_$c.json 2> gpurun_out/r52_$c.err
  python -c "import json;d=json.load(open('gpurun_out/r52_$c.json'));print('$c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['breakdown_ms_per_step'].items()}, round(d['roofline']['frac'],3), d['e2e']['value'], d['device_bytes'])" || tail -5 gpurun_out/r52_$c.err
done
