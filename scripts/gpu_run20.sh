# Round-1 profile refresh: full bench line, reference arm, ncu launch list, one ncu --set full capture of
# every SpMM / GeMM kernel of one training step.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r20_gpu.txt
timeout 900 python bench.py > gpurun_out/r20_bench.json 2> gpurun_out/r20_bench.err; tail -c 600 gpurun_out/r20_bench.json; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r20_ref.json 2> gpurun_out/r20_ref.err; tail -c 300 gpurun_out/r20_ref.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r20_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r20_launches_bench.json 2>&1
python scripts/ncu_launches.py gpurun_out/r20_launches.csv | head -20
# one full step: launches after warm-up (3 steps x 31 kernels per step) -> skip them
timeout 1500 ncu --set full --clock-control none --import-source on --launch-skip 93 --launch-count 31 -o gpurun_out/r20_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r20_full.log 2>&1; tail -2 gpurun_out/r20_full.log
ls -la gpurun_out | tail -5
