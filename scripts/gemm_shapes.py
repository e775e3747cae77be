"""Every tcgen05 GeMM shape of the C4 epoch timed alone (CUDA events, warm, 5 reps), with its fp32 TF/s and
the HBM floor of its operand bytes; `--trace NAME` reruns one shape with the CTA-0 clock trace.
    python scripts/gemm_shapes.py [--trace nn2]"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if "--trace" in sys.argv and "MGGCN_TC_TRACE" not in os.environ:
    os.environ["MGGCN_TC_TRACE"] = "1"
import torch  # noqa: E402  (before libmggcn: torch brings its own NCCL)

from paper_2110_08688_b200 import rowgcn as R  # noqa: E402

for kv in filter(None, os.environ.get("MG_TUNE", "").split(",")):  # e.g. MG_TUNE=gemm_f16=0
    R.set_tuning(kv.split("=")[0], int(kv.split("=")[1]))

M = 2449029
# name: (ta, tb, out rows, out cols, K, epilogue)
SHAPES = {
    "nn0": (False, False, M, 256, 100, 2), "nn1": (False, False, M, 256, 256, 0), "nn2": (False, False, M, 47, 256, 0),
    "nt2": (False, True, M, 256, 47, 1), "nt1": (False, True, M, 256, 256, 1),
    "tn2": (True, False, 256, 47, M, 0), "tn1": (True, False, 256, 256, M, 0), "tn0": (True, False, 100, 256, M, 0),
}


def pad4(d):
    return (d + 3) // 4 * 4


def run(name, reps=5):
    ta, tb, m, n, k, epi = SHAPES[name]
    if ta:  # C[m, n] = A[k, m]^T B[k, n]
        a = torch.randn(k, pad4(m), device="cuda")
        b = torch.randn(k, pad4(n), device="cuda")
        c = torch.empty(8 * m * pad4(n), device="cuda")
        lda, ldb, ldc = pad4(m), pad4(n), pad4(n)
        bytes_ = 4 * k * (m + n)
    else:
        a = torch.randn(m, pad4(k), device="cuda")
        b = torch.randn(n, pad4(k), device="cuda") if tb else torch.randn(k, pad4(n), device="cuda")
        c = torch.randn(m, pad4(n), device="cuda")
        lda, ldb, ldc = pad4(k), pad4(k) if tb else pad4(n), pad4(n)
        bytes_ = 4 * m * (k + n * (2 if epi == 1 else 1))
    args = (ta, tb, m, n, k, a.data_ptr(), lda, b.data_ptr(), ldb, c.data_ptr(), ldc, epi, R.GEMM_TF32X3)
    R.dev_gemm(*args)
    torch.cuda.synchronize()
    if os.environ.get("MGGCN_TC_TRACE"):
        return
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        R.dev_gemm(*args)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    flops = 2.0 * m * n * k
    print(f"{name}: {ms:.3f} ms  {flops / ms / 1e9:.0f} fp32 TF/s  HBM floor {bytes_ / 6.55e9:.3f} ms")


if __name__ == "__main__":
    if "--trace" in sys.argv:
        run(sys.argv[sys.argv.index("--trace") + 1])
    elif "--only" in sys.argv:
        run(sys.argv[sys.argv.index("--only") + 1], reps=1)
    else:
        for nm in SHAPES:
            run(nm)
