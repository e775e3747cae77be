cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 120 python scripts/gemm_trace.py 3 2>&1 | grep -E "err|s1[0-9] |s2[0-9] |acc" | head -30
timeout 300 python -c "
import sys; sys.path.insert(0, '.')
import torch, pytest
from paper_2110_08688_b200 import rowgcn as R
R.set_tuning('gemm_kernel', 3)
sys.exit(pytest.main(['tests/test_gpu_kernels.py', 'tests/test_gpu_model.py', '-q', '-x', '-p', 'no:cacheprovider']))
" 2>&1 | tail -3
for k in 2 3; do timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --gemm-kernel $k 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('kernel $k', round(d['ms_per_step'],2), d['breakdown_ms_per_step'])"; done
