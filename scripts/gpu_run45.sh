# SpMM hub-hint footprint sweep, interleaved on one box.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in 1 2; do for hb in 100663296 67108864 134217728 50331648; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --spmm-hub-bytes $hb 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);b=d['breakdown_ms_per_step'];print('hub $hb', round(d['ms_per_step'],2), 'spmm', round(b['spmm'],3))"
done; done
