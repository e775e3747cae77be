cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export MGGCN_TC_TRACE=1
timeout 120 python -c "
import os, sys; sys.path.insert(0, '.')
from paper_2110_08688_b200 import rowgcn as R
R.set_tuning('gemm_kernel', 3)
exec(open('scripts/gemm_trace.py').read().split('os.environ[\"MGGCN_TC_TRACE\"] = \"1\"')[1])
" 2>&1 | tail -40
unset MGGCN_TC_TRACE
timeout 300 python -c "
import sys; sys.path.insert(0, '.')
import pytest
from paper_2110_08688_b200 import rowgcn as R
R.set_tuning('gemm_kernel', 3)
sys.exit(pytest.main(['tests/test_gpu_kernels.py', '-q', '-x', '-p', 'no:cacheprovider', '-k', 'tc or tf32 or gemm']))
" 2>&1 | tail -3
for k in 2 3; do timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --gemm-kernel $k 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('kernel $k', round(d['ms_per_step'],2), d['breakdown_ms_per_step'])"; done
