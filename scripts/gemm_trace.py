"""One NN tcgen05 GeMM at C4 layer-1 shape with the CTA-0 clock trace (MGGCN_TC_TRACE=1).
    python scripts/gemm_trace.py [gemm_kernel]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402  (before libmggcn: torch brings its own NCCL)
os.environ["MGGCN_TC_TRACE"] = "1"
from paper_2110_08688_b200 import rowgcn as R  # noqa: E402
if len(sys.argv) > 1:
    R.set_tuning("gemm_kernel", int(sys.argv[1]))
M, K, N = 2449029, 256, 256
a = torch.randn(M, K, device="cuda")
w = torch.randn(K, N, device="cuda")
c = torch.empty(M, N, device="cuda")
for _ in range(2):
    R.dev_gemm(False, False, M, N, K, a.data_ptr(), K, w.data_ptr(), N, c.data_ptr(), N, 0, R.GEMM_TF32X3)
torch.cuda.synchronize()
ref = (a[:4096].double() @ w.double()).float()
print("max rel err (first 4096 rows):", float((c[:4096] - ref).abs().max() / ref.abs().max()))

# TN (W-grad) at the C4 layer-1 shape: H^T G over 8 canonical blocks of the rows
h = torch.randn(M, 256, device="cuda")
g = torch.randn(M, 256, device="cuda")
stage = torch.empty(8 * 256 * 256, device="cuda")
import ctypes as C  # noqa: E402
for _ in range(2):
    R.dev_gemm(True, False, 256, 256, M, h.data_ptr(), 256, g.data_ptr(), 256, stage.data_ptr(), 256, 0,
               R.GEMM_TF32X3)
torch.cuda.synchronize()
