"""GPU diagnostic: accuracy of the tcgen05 3xTF32 GeMMs (normwise and per-column bias) on the shapes and value
distributions of the C4 step, and of the products 1/16 sample's teacher-forced step under mode combinations.

  python scripts/gemm_bias_probe.py [gemm] [step]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import torch  # noqa: E402

from paper_2110_08688_b200 import rowgcn as R  # noqa: E402
from gpu_util import dev_padded, normwise  # noqa: E402


def run_gemm(a, b, ta, tb, mode, epi=0, c0=None):
    m = a.shape[1] if ta else a.shape[0]
    k = a.shape[0] if ta else a.shape[1]
    n = b.shape[0] if tb else b.shape[1]
    a_d, b_d = dev_padded(a), dev_padded(b)
    c_d = dev_padded(c0 if c0 is not None else np.zeros((m, n), np.float32))
    R.dev_gemm(ta, tb, m, n, k, a_d.data_ptr(), a_d.shape[1], b_d.data_ptr(), b_d.shape[1], c_d.data_ptr(),
               c_d.shape[1], epi, mode)
    torch.cuda.synchronize()
    return c_d.cpu().numpy()[:, :n]


def bias(got, ref):
    """max over columns of |sum(got - ref)| / sum|ref| (coherent error)"""
    d = (got.astype(np.float64) - ref).sum(0)
    return float(np.max(np.abs(d) / np.maximum(np.abs(ref).sum(0), 1e-30)))


def gemm_probe():
    rng = np.random.default_rng(0)
    dists = {"sym": lambda s: rng.uniform(-1, 1, s), "pos": lambda s: rng.uniform(0, 1, s),
             "relu_gauss": lambda s: np.maximum(rng.normal(size=s), 0), "tiny": lambda s: rng.normal(size=s) * 1e-6}
    cases = [("NN", False, False, 20000, 256, 100), ("NN", False, False, 20000, 256, 256),
             ("NT", False, True, 20000, 256, 47), ("NT", False, True, 20000, 256, 256),
             ("TN", True, False, 256, 256, 153000), ("TN", True, False, 100, 256, 306000),
             ("TN", True, False, 256, 48, 306000)]
    out = []
    rn = "MG_TC_SPLIT_RN (compile time)"
    if True:
        for name, ta, tb, m, n, k in cases:
            for da, db in (("sym", "sym"), ("relu_gauss", "sym"), ("pos", "pos"), ("relu_gauss", "tiny")):
                a = dists[da]((k, m) if ta else (m, k)).astype(np.float32)
                b = dists[db]((n, k) if tb else (k, n)).astype(np.float32)
                ref = (a.astype(np.float64).T if ta else a.astype(np.float64)) @ (b.astype(np.float64).T if tb else b)
                got = run_gemm(a, b, ta, tb, R.GEMM_TF32X3)
                r = dict(rn=rn, op=name, m=m, n=n, k=k, a=da, b=db, normwise=normwise(got, ref), bias=bias(got, ref))
                # the fp32 serial reference's own error (k-ascending fold) for scale, on the small cases
                print(json.dumps(r), flush=True)
                out.append(r)
    return out


def step_probe():
    import test_gpu_scale as T
    fx = np.load(os.path.join(ROOT, "tests", "golden", "scale_c4s16step.npz"))
    variants = {
        "prod": dict(gemm_mode=R.GEMM_TF32X3, spmm_mode=R.SPMM_FAST, aggregate_input=True),
        "tc_exactspmm": dict(gemm_mode=R.GEMM_TF32X3, spmm_mode=R.SPMM_EXACT, aggregate_input=True),
        "exactgemm_fast": dict(gemm_mode=R.GEMM_EXACT, spmm_mode=R.SPMM_FAST, aggregate_input=True),
        "prod_noagg": dict(gemm_mode=R.GEMM_TF32X3, spmm_mode=R.SPMM_FAST, aggregate_input=False),
    }
    rn = "MG_TC_SPLIT_RN (compile time)"
    if True:
        for name, mode in variants.items():
            T.MODES["probe"] = mode
            ours = T.teacher_forced_dump("c4s16", "probe", 1)
            rep = {}
            for key in ["fwd0", "fwd1", "fwd2", "loss_grad", "bwd0", "bwd1"]:
                rep[key] = [round(x, 8) for x in T.check_rows(ours[key], fx, key)]
            for l in range(3):
                rep[f"wgrad{l}"] = round(normwise(ours[f"wgrad{l}"], fx[f"wgrad{l}"]), 8)
            print(json.dumps(dict(rn=rn, variant=name, **rep)), flush=True)


if __name__ == "__main__":
    what = sys.argv[1:] or ["gemm", "step"]
    if "gemm" in what:
        gemm_probe()
    if "step" in what:
        step_probe()
