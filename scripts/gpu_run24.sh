cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
b() { tag=$1; shift; timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/b24_$tag.json 2> gpurun_out/b24_$tag.err
  python -c "import json;d=json.load(open('gpurun_out/b24_$tag.json'));print('$tag', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['breakdown_ms_per_step'].items()})" || tail -5 gpurun_out/b24_$tag.err; }
b h0 --spmm-hub-bytes 0
for mb in 32 48 72 96 128; do b h$mb --spmm-hub-bytes $((mb << 20)); done
