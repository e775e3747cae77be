cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tuning.py -q -p no:cacheprovider 2>&1 | tail -3
for g in 0 4 8; do
  timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --spmm-narrow-group $g > gpurun_out/bench12_g$g.json 2> gpurun_out/bench12_g$g.err
  python -c "import json;d=json.load(open('gpurun_out/bench12_g$g.json'));print('group $g', round(d['ms_per_step'],2), d['breakdown_ms_per_step'], round(d['roofline']['frac'],3))" || tail -3 gpurun_out/bench12_g$g.err
done
