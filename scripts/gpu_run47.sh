# ncu source-level (SASS) stall sampling of one TN W-grad GeMM at the C4 layer-1 shape.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:"gemm_tc2" --launch-skip 1 --launch-count 1 -o gpurun_out/r47_tn1 -f python scripts/gemm_shapes.py --only tn1 > gpurun_out/r42.log 2>&1; tail -2 gpurun_out/r42.log
ncu -i gpurun_out/r47_tn1.ncu-rep --page source --csv --print-source sass > gpurun_out/r47_tn1_sass.csv 2>&1; wc -l gpurun_out/r47_tn1_sass.csv
rm -f gpurun_out/r47_tn1.ncu-rep
