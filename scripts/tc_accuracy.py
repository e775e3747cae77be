"""Accuracy probe of the tcgen05 kind::tf32 GeMMs (GPU): normwise error and mean signed error (bias)
against an fp64 product, as a function of the reduction length K and of the TN split-K chunk.
Run on the GPU box: python scripts/tc_accuracy.py > gpurun_out/tc_accuracy.txt"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from gpu_util import dev_padded  # noqa: E402

from paper_2110_08688_b200 import rowgcn as R  # noqa: E402


def run(a, b, ta, tb, mode):
    m = a.shape[1] if ta else a.shape[0]
    k = a.shape[0] if ta else a.shape[1]
    n = b.shape[0] if tb else b.shape[1]
    a_d, b_d = dev_padded(a), dev_padded(b)
    c_d = dev_padded(np.zeros((m, n), np.float32))
    R.dev_gemm(ta, tb, m, n, k, a_d.data_ptr(), a_d.shape[1], b_d.data_ptr(), b_d.shape[1], c_d.data_ptr(),
               c_d.shape[1], 0, mode)
    torch.cuda.synchronize()
    return c_d.cpu().numpy()[:, :n]


def stats(got, ref):
    d = got.astype(np.float64) - ref
    sgn = np.sign(ref)
    return np.max(np.abs(d)) / np.max(np.abs(ref)), float(np.mean(d * sgn) / np.mean(np.abs(ref)))


rng = np.random.default_rng(0)
print("mode K normwise bias(rel, + = away from zero)")
for mode, name in ((R.GEMM_TF32X3, "tf32x3"), (R.GEMM_TF32, "tf32")):
    for K in (64, 256, 1024, 4096):
        a = rng.uniform(-1, 1, (2048, K)).astype(np.float32)
        b = rng.uniform(-1, 1, (K, 256)).astype(np.float32)
        ref = a.astype(np.float64) @ b
        print("NN", name, K, *stats(run(a, b, False, False, mode), ref))
    for chunk in (256, 1024, 4096, 16384):
        R.set_tuning("tn_chunk", chunk)
        a = rng.uniform(-1, 1, (65536, 256)).astype(np.float32)
        b = rng.uniform(-1, 1, (65536, 256)).astype(np.float32)
        ref = a.astype(np.float64).T @ b
        print("TN", name, "chunk", chunk, *stats(run(a, b, True, False, mode), ref))
    R.set_tuning("tn_chunk", 4096)
# positive-only inputs expose a truncating accumulator as a one-sided bias
a = rng.uniform(0, 1, (65536, 128)).astype(np.float32)
b = rng.uniform(0, 1, (65536, 128)).astype(np.float32)
ref = a.astype(np.float64).T @ b
for chunk in (256, 4096):
    R.set_tuning("tn_chunk", chunk)
    print("TN positive tf32x3 chunk", chunk, *stats(run(a, b, True, False, R.GEMM_TF32X3), ref))
R.set_tuning("tn_chunk", 4096)
