cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 120 python -c "
import sys, os; sys.path.insert(0, '.')
import torch, numpy as np
from paper_2110_08688_b200 import rowgcn as R
R.set_tuning('gemm_kernel', 4)
M, K, N = 1000, 256, 256
a = torch.randn(M, K, device='cuda'); w = torch.randn(K, N, device='cuda'); c = torch.zeros(M, N, device='cuda')
R.dev_gemm(False, False, M, N, K, a.data_ptr(), K, w.data_ptr(), N, c.data_ptr(), N, 0, R.GEMM_TF32X3)
torch.cuda.synchronize()
ref = (a.double() @ w.double())
print('v4 small err', float((c.double() - ref).abs().max() / ref.abs().max()))
" 2>&1 | tail -3
echo "rc=$?"
timeout 300 python -c "
import sys; sys.path.insert(0, '.')
import torch, pytest
from paper_2110_08688_b200 import rowgcn as R
R.set_tuning('gemm_kernel', 4)
sys.exit(pytest.main(['tests/test_gpu_kernels.py', '-q', '-x', '-p', 'no:cacheprovider', '-k', 'tcgen05 and kernel3']))
" 2>&1 | tail -3
for k in 3 4; do timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --gemm-kernel $k 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('kernel $k', round(d['ms_per_step'],2), d['breakdown_ms_per_step'])"; done
