#!/usr/bin/env bash
# C4 step A/B of the W-grad split-K chunk (tn_chunk 4096 default vs 8192), alternating, three rounds
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
for r in 1 2 3; do for c in 4096 8192; do
  timeout 600 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-cold-e2e --no-ax-extra --tune tn_chunk=$c > gpurun_out/tnc.json 2> gpurun_out/tnc.err
  python -c "import json;d=json.load(open('gpurun_out/tnc.json'));print('tn_chunk=$c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['breakdown_ms_per_step'].items()}, d['clocks']['sm_mhz'], round(d['loss'],7))" || tail -3 gpurun_out/tnc.err
done; done
