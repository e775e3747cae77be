#!/usr/bin/env bash
# v3 NN / NT epilogue-buffer / W-ring A/B on the C4 GeMM shapes (scripts/gemm_shapes.py), two rounds each
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
O=gpurun_out/epi_probe.txt; : > $O
for r in 1 2; do
  for t in "" "gemm3_epi=4" "gemm3_epi=4,gemm3_wring=65536" "gemm3_epi=1"; do
    echo "== round $r tune '$t'" >> $O
    MG_TUNE=$t python scripts/gemm_shapes.py 2>&1 | grep -E "^nn|^nt" >> $O
  done
done
cat $O
