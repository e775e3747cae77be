"""Debug probe for the tcgen05 GeMM (run with MGGCN_TC_DEBUG=1 on the GPU box)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from gpu_util import dev_padded  # noqa: E402

from paper_2110_08688_b200 import rowgcn as R  # noqa: E402

for (m, n, k, tb) in [(128, 32, 16, False), (128, 32, 16, True), (256, 64, 48, False)]:
    a = (np.arange(m * k, dtype=np.float32).reshape(m, k) % 7 + 1) / 8
    b = (np.arange(n * k, dtype=np.float32).reshape((n, k) if tb else (k, n)) % 5 + 1) / 4
    ref = a.astype(np.float64) @ (b.T if tb else b)
    for mode in (R.GEMM_TF32, R.GEMM_TF32X3):
        a_d, b_d = dev_padded(a), dev_padded(b)
        c_d = dev_padded(np.zeros((m, n), np.float32))
        R.dev_gemm(False, tb, m, n, k, a_d.data_ptr(), a_d.shape[1], b_d.data_ptr(), b_d.shape[1], c_d.data_ptr(),
                   c_d.shape[1], 0, mode)
        torch.cuda.synchronize()
        got = c_d.cpu().numpy()[:, :n]
        print(f"m={m} n={n} k={k} tb={tb} mode={mode}: max|d|={np.max(np.abs(got - ref)):.3g} "
              f"ref[0,:4]={ref[0, :4]} got[0,:4]={got[0, :4]}", flush=True)
        print("   a[0,:8]", a[0, :8], " b[0,:8]", b[0, :8], flush=True)

# TN (both operands MN-major)
for (m, n, k) in [(128, 32, 16), (128, 64, 300), (256, 48, 5000)]:
    a = (np.arange(k * m, dtype=np.float32).reshape(k, m) % 7 + 1) / 8
    b = (np.arange(k * n, dtype=np.float32).reshape(k, n) % 5 + 1) / 4
    ref = a.astype(np.float64).T @ b
    for mode in (R.GEMM_TF32, R.GEMM_TF32X3):
        a_d, b_d = dev_padded(a), dev_padded(b)
        c_d = dev_padded(np.zeros((m, n), np.float32))
        R.dev_gemm(True, False, m, n, k, a_d.data_ptr(), a_d.shape[1], b_d.data_ptr(), b_d.shape[1], c_d.data_ptr(),
                   c_d.shape[1], 0, mode)
        torch.cuda.synchronize()
        got = c_d.cpu().numpy()[:, :n]
        print(f"TN m={m} n={n} k={k} mode={mode}: max rel|d|={np.max(np.abs(got - ref)) / np.max(np.abs(ref)):.3g}",
              flush=True)
