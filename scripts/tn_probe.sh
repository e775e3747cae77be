#!/usr/bin/env bash
# W-grad TN probe: every GeMM shape of the C4 epoch timed alone, CTA-0 clock traces of the TN /
# NT shapes, and the TN split-K chunk (tn_chunk) swept.  gpurun --timeout 900 -- 'bash scripts/tn_probe.sh'
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python scripts/gemm_shapes.py > gpurun_out/tn_shapes.txt 2>&1
for s in tn1 tn0 nt2; do python scripts/gemm_shapes.py --trace $s > gpurun_out/tn_trace_$s.txt 2>&1; done
for c in 2048 8192 16384; do echo "tn_chunk=$c" >> gpurun_out/tn_shapes.txt; MG_TUNE=tn_chunk=$c python scripts/gemm_shapes.py --only tn1 >> gpurun_out/tn_shapes.txt 2>&1; done
