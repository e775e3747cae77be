# Half-size tc3 epilogue buffers + W ring sweep; GeMM parity first.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_properties.py tests/test_gpu_model.py tests/test_gpu_flags.py tests/test_gpu_tuning.py -q -x -p no:cacheprovider 2>&1 | tail -2
for w in 65536 98304 131072; do timeout 300 python - <<EOF2 2>&1 | tail -1
import sys, json, io, contextlib, runpy
sys.argv = ["bench.py", "--steps", "10", "--warmup", "3", "--no-cpu-baseline", "--no-e2e"]
import torch
from paper_2110_08688_b200 import rowgcn as R
R.set_tuning("gemm3_wring", $w)
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    runpy.run_path("bench.py", run_name="__main__")
d = json.loads(buf.getvalue().strip().splitlines()[-1])
print("wring $w", round(d["ms_per_step"], 2), d["breakdown_ms_per_step"])
EOF2
done
