#!/usr/bin/env bash
# One parameterised GPU-box runner (replaces the round-1 one-off gpu_runNN.sh scripts).
#   gpurun --timeout S -- 'bash scripts/gpu_run.sh TAG task [task ...]'
# Every output lands in gpurun_out/TAG_*. Tasks:
#   suite            pytest -m gpu + smoke()
#   tests:EXPR       pytest -m gpu -k EXPR
#   bench            default bench line (C4, e2e, cpu baseline) + the reference arm
#   cfg:NAME         bench line of another config (c1 c2 c3 c5s ...), no cpu baseline
#   launches         ncu launch list (gpu__time_duration) of a 2-step C4 bench
#   ncu_spmm[:CFG]   ncu --set full of 10 SpMM launches of one step, summarised
#   ncu_gemm[:CFG]   ncu --set full of the GeMM / loss launches of one step, summarised
#   py:SCRIPT        python SCRIPT (extra args via GPU_RUN_ARGS)
set -u
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
TAG=$1; shift
O=gpurun_out/$TAG
for task in "$@"; do
  name=${task%%:*}; arg=${task#*:}; [ "$arg" = "$task" ] && arg=""
  echo "== $task"
  case $name in
    suite)
      timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > ${O}_pytest.log 2>&1; tail -3 ${O}_pytest.log
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.log 2>&1; tail -2 ${O}_smoke.log ;;
    tests)
      timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -k "$arg" > ${O}_tests.log 2>&1; tail -15 ${O}_tests.log ;;
    bench)
      timeout 900 python bench.py > ${O}_bench.json 2> ${O}_bench.err; tail -c 600 ${O}_bench.json; echo
      timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > ${O}_ref.json 2> ${O}_ref.err; tail -c 300 ${O}_ref.json; echo ;;
    cfg)
      timeout 1200 python bench.py --config $arg --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} > ${O}_$arg.json 2> ${O}_$arg.err
      python -c "import json;d=json.load(open('${O}_$arg.json'));print('$arg', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['breakdown_ms_per_step'].items()}, round(d['roofline']['frac'],3), (d['e2e'] or {}).get('value'), d['device_bytes'])" || tail -5 ${O}_$arg.err ;;
    launches)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${O}_launches.csv python bench.py --config ${arg:-c4} --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > ${O}_launches_bench.json 2>&1
      python scripts/ncu_launches.py ${O}_launches.csv > ${O}_launches.txt; head -16 ${O}_launches.txt ;;
    ncu_spmm)
      # every SpMM launch of ONE step (ncu flushes caches between kernels, so no warm-up is needed)
      c=${arg:-c4}
      timeout 2400 ncu --set full --clock-control none --import-source on -k regex:"spmm_" -o ${O}_spmm_$c -f python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > ${O}_spmm_$c.log 2>&1; tail -1 ${O}_spmm_$c.log
      ncu -i ${O}_spmm_$c.ncu-rep --page raw --csv > ${O}_spmm_${c}_raw.csv 2>&1
      python scripts/ncu_summary.py ${O}_spmm_$c.ncu-rep > ${O}_ncu_spmm_$c.txt 2>&1; head -30 ${O}_ncu_spmm_$c.txt
      [ -n "${KEEP_REP:-}" ] || rm -f ${O}_spmm_$c.ncu-rep ;;
    ncu_gemm)
      timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc|softmax" --launch-skip ${NCU_SKIP:-27} --launch-count ${NCU_COUNT:-9} -o ${O}_gemm -f python bench.py --config ${arg:-c4} --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > ${O}_gemm.log 2>&1; tail -1 ${O}_gemm.log
      python scripts/ncu_summary.py ${O}_gemm.ncu-rep > ${O}_ncu_gemm.txt 2>&1; head -30 ${O}_ncu_gemm.txt; rm -f ${O}_gemm.ncu-rep ;;
    py)
      timeout 1800 python $arg ${GPU_RUN_ARGS:-} > ${O}_py.log 2>&1; tail -40 ${O}_py.log ;;
    *) echo "unknown task $task" ;;
  esac
done
