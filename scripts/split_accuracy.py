"""CPU simulation of the operand splits for fp32 GeMMs on tensor cores (products exact, fp64 sums):
3xTF32 (hi = x & 0xFFFFE000, lo = x - hi, tf32-truncated) against a two-term fp16 split with a per-tensor
power-of-two scale (hi = fp16(s x), lo = fp16(s x - hi)), on activation-like and gradient-like inputs.
    python scripts/split_accuracy.py"""
import numpy as np


def tf32(x):
    return (x.astype(np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


def split_tf32(x):
    hi = tf32(x)
    lo = tf32(x - hi)  # the tensor core reads lo truncated to tf32 as well
    return hi.astype(np.float64), lo.astype(np.float64)


def split_f16(x):
    m = np.abs(x).max()
    e = np.floor(np.log2(m)) if m > 0 else 0
    s = 2.0 ** (14 - e)  # max |s x| in [2^14, 2^15)
    xs = (x.astype(np.float64) * s)
    hi = xs.astype(np.float16)
    lo = (xs - hi.astype(np.float64)).astype(np.float16)
    return hi.astype(np.float64) / s, lo.astype(np.float64) / s


def gemm3(a, b, split):
    ah, al = split(a)
    bh, bl = split(b)
    return ah @ bh + ah @ bl + al @ bh


def normwise(x, ref):
    return float(np.abs(x - ref).max() / np.abs(ref).max())


rng = np.random.default_rng(0)
K, M, N = 256, 4096, 256
cases = {
    "uniform(-1,1)": (rng.uniform(-1, 1, (M, K)), rng.uniform(-1, 1, (K, N))),
    "relu activations x glorot W": (np.maximum(rng.normal(0, 1, (M, K)), 0), rng.uniform(-0.15, 0.15, (K, N))),
    "gradients ~1e-7 x glorot W": (rng.normal(0, 1e-7, (M, K)), rng.uniform(-0.15, 0.15, (K, N))),
    "heavy-tailed (lognormal)": (rng.lognormal(0, 3, (M, K)) * rng.choice([-1, 1], (M, K)), rng.uniform(-1, 1, (K, N))),
}
print(f"{'inputs':32s} {'3xTF32':>10s} {'f16 x2 (scaled)':>16s}")
for name, (a, b) in cases.items():
    a = a.astype(np.float32)
    b = b.astype(np.float32)
    ref = a.astype(np.float64) @ b.astype(np.float64)
    print(f"{name:32s} {normwise(gemm3(a, b, split_tf32), ref):10.2e} {normwise(gemm3(a, b, split_f16), ref):16.2e}")
