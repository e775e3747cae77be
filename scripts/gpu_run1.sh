set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -40 > gpurun_out/pytest1.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke1.log 2>&1
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err
tail -5 gpurun_out/pytest1.log; cat gpurun_out/smoke1.log; cat gpurun_out/bench1.json; tail -5 gpurun_out/bench1.err
