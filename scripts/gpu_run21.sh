cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tuning.py -q -p no:cacheprovider -x -k async 2>&1 | tail -4
b() { tag=$1; shift; timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/b21_$tag.json 2> gpurun_out/b21_$tag.err
  python -c "import json;d=json.load(open('gpurun_out/b21_$tag.json'));print('$tag', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['breakdown_ms_per_step'].items()})" || tail -5 gpurun_out/b21_$tag.err; }
b async
b sync --spmm-async 0
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/r21_launches.csv -k regex:spmm python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/r21_launches.csv')) if len(r)>10]
hdr=rows[0]
for r in rows[1:]:
    d=dict(zip(hdr,r))
    print(d['Kernel Name'][:40], d['Metric Name'], d['Metric Value'])
PY
