# A/B of two builds of libmggcn.so on one box: _ab/lib_A.so and _ab/lib_B.so, interleaved C4 benches.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cp paper_2110_08688_b200/libmggcn.so _ab/lib_orig.so
for i in $(seq ${AB_REPS:-3}); do for v in A B; do
  cp _ab/lib_$v.so paper_2110_08688_b200/libmggcn.so
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${AB_EXTRA:---no-e2e} 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);b=d['breakdown_ms_per_step'];print('$v', (d['e2e'] or {}).get('value'), d['loss'], round(d['ms_per_step'],2), 'spmm', round(b['spmm'],2), 'gemm', round(b['gemm'],3), 'other', round(b['other'],3))"
done; done
cp _ab/lib_orig.so paper_2110_08688_b200/libmggcn.so
