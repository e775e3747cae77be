"""GPU parity of the sm_100a kernels through the C ABI (mg_dev_spmm / mg_dev_gemm) against the CPU
oracles: exact modes must be BITWISE equal to the reference's f32 arithmetic (inc/sparse.hpp:144-153,
inc/dense.hpp:140-204)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
from gpu_util import bits_equal, dev_padded, dev_tile, pad4  # noqa: E402

from paper_2110_08688_b200 import rowgcn as R  # noqa: E402


def run_spmm(rp, ci, v, h, accumulate=False, out0=None, relu=False, mode=R.SPMM_EXACT):
    rows = len(rp) - 1
    w = h.shape[1]
    ld = pad4(w)
    rp_d, ed_d = dev_tile(rp, ci, v)
    h_d = dev_padded(h, ld)
    out_d = dev_padded(out0 if out0 is not None else np.zeros((rows, w), np.float32), ld)
    R.dev_spmm(rows, rp_d.data_ptr(), ed_d.data_ptr(), h_d.data_ptr(), out_d.data_ptr(), w, ld, accumulate, relu, mode)
    torch.cuda.synchronize()
    out = out_d.cpu().numpy()
    assert np.all(out[:, w:] == 0), "padding columns must stay zero"
    return out[:, :w]


@pytest.mark.parametrize("k", range(4))
def test_spmm_exact_golden(golden, k):
    rp, ci, v = golden[f"spmm{k}_f32_rp"], golden[f"spmm{k}_f32_ci"], golden[f"spmm{k}_f32_v"]
    h = golden[f"spmm{k}_f32_h"]
    assert bits_equal(run_spmm(rp, ci, v, h), golden[f"spmm{k}_f32_out"])
    out = run_spmm(rp, ci, v, h, accumulate=True, out0=golden[f"spmm{k}_f32_o0"])
    assert bits_equal(out, golden[f"spmm{k}_f32_acc"])


def random_tile(rng, rows, cols, density, hub_rows=(), hub_len=0):
    rp = [0]
    ci, v = [], []
    for r in range(rows):
        if r in hub_rows:
            cols_r = np.sort(rng.choice(cols, size=min(hub_len, cols), replace=False))
        else:
            cols_r = np.nonzero(rng.random(cols) < density)[0]
        ci.extend(cols_r.tolist())
        v.extend(rng.uniform(-1, 1, len(cols_r)).tolist())
        rp.append(len(ci))
    return np.array(rp, np.int64), np.array(ci, np.int64), np.array(v, np.float32)


@pytest.mark.parametrize("w", [1, 3, 4, 7, 16, 40, 47, 64, 128, 256, 300, 602, 1100])
def test_spmm_exact_widths(port32, w):
    rng = np.random.default_rng(w)
    rows, cols = 150, 90
    rp, ci, v = random_tile(rng, rows, cols, 0.08)
    h = rng.uniform(-1, 1, (cols, w)).astype(np.float32)
    ref = port32.spmm(rows, cols, rp, ci, v, h)
    assert bits_equal(run_spmm(rp, ci, v, h), ref)
    o0 = rng.uniform(-1, 1, (rows, w)).astype(np.float32)
    ref_acc = port32.spmm(rows, cols, rp, ci, v, h, True, o0)
    assert bits_equal(run_spmm(rp, ci, v, h, True, o0), ref_acc)
    relu = run_spmm(rp, ci, v, h, True, o0, relu=True)
    assert bits_equal(relu, np.where(ref_acc > 0, ref_acc, np.float32(0)))


@pytest.mark.parametrize("w", [8, 48, 256])
def test_spmm_exact_hub_rows(port32, w):
    """Rows above the heavy threshold take the cp.async hub kernel; still bitwise exact."""
    rng = np.random.default_rng(7 + w)
    rows, cols = 300, 5000
    rp, ci, v = random_tile(rng, rows, cols, 0.002, hub_rows=(0, 17, 299), hub_len=4500)
    h = rng.uniform(-1, 1, (cols, w)).astype(np.float32)
    o0 = rng.uniform(-1, 1, (rows, w)).astype(np.float32)
    ref = port32.spmm(rows, cols, rp, ci, v, h, True, o0)
    R.set_tuning("heavy_row", 1000)
    try:
        out = run_spmm(rp, ci, v, h, True, o0)
    finally:
        R.set_tuning("heavy_row", 4096)
    assert bits_equal(out, ref)


def test_spmm_empty_rows_and_tile():
    rp = np.zeros(6, np.int64)
    out = run_spmm(rp, np.zeros(0, np.int64), np.zeros(0, np.float32), np.ones((4, 5), np.float32))
    assert np.all(out == 0)


def run_gemm(a, b, ta, tb, epi=0, c0=None, mode=R.GEMM_EXACT):
    m = a.shape[1] if ta else a.shape[0]
    k = a.shape[0] if ta else a.shape[1]
    n = b.shape[0] if tb else b.shape[1]
    a_d = dev_padded(a)
    b_d = dev_padded(b)
    c_d = dev_padded(c0 if c0 is not None else np.zeros((m, n), np.float32))
    R.dev_gemm(ta, tb, m, n, k, a_d.data_ptr(), a_d.shape[1], b_d.data_ptr(), b_d.shape[1], c_d.data_ptr(),
               c_d.shape[1], epi, mode)
    torch.cuda.synchronize()
    return c_d.cpu().numpy()[:, :n]


@pytest.mark.parametrize("k,ta,tb", [(0, False, False), (1, True, False), (2, False, True)])
def test_gemm_exact_golden(golden, k, ta, tb):
    a, b = golden[f"gemm{k}_f32_a"], golden[f"gemm{k}_f32_b"]
    assert bits_equal(run_gemm(a, b, ta, tb), golden[f"gemm{k}_f32_out"])


@pytest.mark.parametrize("shape", [(1, 1, 1), (70, 33, 65), (300, 256, 100), (129, 47, 256), (5, 300, 17)])
@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True)])
def test_gemm_exact_shapes(port32, shape, ta, tb):
    m, n, k = shape
    rng = np.random.default_rng(m * 7 + n * 3 + k)
    a = rng.uniform(-1, 1, (k, m) if ta else (m, k)).astype(np.float32)
    a[rng.random(a.shape) < 0.3] = 0
    b = rng.uniform(-1, 1, (n, k) if tb else (k, n)).astype(np.float32)
    ref = port32.gemm(a, b, ta, tb)
    assert bits_equal(run_gemm(a, b, ta, tb), ref)
    if not ta:
        c0 = rng.normal(size=(m, n)).astype(np.float32)
        got = run_gemm(a, b, ta, tb, epi=1, c0=c0)  # relu_backward mask (dense.hpp:221-231)
        assert bits_equal(got, np.where(c0 > 0, ref, np.float32(0)))
        got = run_gemm(a, b, ta, tb, epi=2)
        assert bits_equal(got, np.where(ref > 0, ref, np.float32(0)))


# ---------------------------------------------------------------------------- tcgen05 GeMMs
# TF32X3 (3-term hi/lo split on kind::tf32): normwise error vs an fp64 product <= 1e-5 (measured ~1e-6);
# TF32 (1 term) is the reduced-precision mode and only has to be within 5e-3.
TC_SHAPES = [(1000, 256, 100), (777, 256, 256), (130, 48, 256), (300, 256, 47), (64, 16, 8), (513, 100, 602),
             (2000, 256, 33)]


@pytest.mark.parametrize("mode,tol", [(R.GEMM_TF32X3, 1e-5), (R.GEMM_TF32, 5e-3)])
@pytest.mark.parametrize("shape", TC_SHAPES)
@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False)])
# 1: both operands split in smem (SS); 2: A split into TMEM (TS); 3 (default): 2 with 32-K SWIZZLE_128B stages
# and decoupled A / W rings for NN / NT (TN runs the v2 kernel under 3), NN / NT on the scaled fp16 two-term
# split (kind::f16, per-row A / per-column W power-of-two scales); 30: 3 with the 3xTF32 split for NN / NT
@pytest.mark.parametrize("kernel", [1, 2, 3, 30])
def test_gemm_tcgen05(gemm_kernel, shape, ta, tb, mode, tol):
    from gpu_util import normwise
    m, n, k = shape
    if ta:  # W-grad shape: M, N = layer widths, K = rows (exercise several 4096-row split-K chunks)
        m, n, k = min(m, 256), n, k * 23
    rng = np.random.default_rng(m + 3 * n + 7 * k + 11 * ta + 13 * tb)
    a = rng.uniform(-1, 1, (k, m) if ta else (m, k)).astype(np.float32)
    b = rng.uniform(-1, 1, (n, k) if tb else (k, n)).astype(np.float32)
    ref = (a.astype(np.float64).T if ta else a.astype(np.float64)) @ (b.astype(np.float64).T if tb else b)
    got = run_gemm(a, b, ta, tb, mode=mode)
    assert normwise(got, ref) <= tol, normwise(got, ref)
    if not ta:
        c0 = rng.normal(size=(m, n)).astype(np.float32)
        got1 = run_gemm(a, b, ta, tb, epi=1, c0=c0, mode=mode)
        assert np.all(got1[c0 <= 0] == 0)
        assert normwise(got1, np.where(c0 > 0, ref, 0)) <= tol
        got2 = run_gemm(a, b, ta, tb, epi=2, mode=mode)
        assert np.all(got2 >= 0) and normwise(got2, np.maximum(ref, 0)) <= tol


@pytest.fixture
def gemm_kernel(kernel):
    R.set_tuning("gemm_kernel", 3 if kernel == 30 else kernel)
    R.set_tuning("gemm_f16", 0 if kernel == 30 else 1)
    R.set_tuning("gemm_f16_min_k", 0)  # the fp16 split at every K (the step uses it above K = 128)
    yield kernel
    R.set_tuning("gemm_kernel", 3)
    R.set_tuning("gemm_f16", 0)
    R.set_tuning("gemm_f16_min_k", 128)


# Scaled fp16 split (kernel 3, NN / NT): rows and columns of very different magnitudes, tiny (gradient-like)
# and huge values, zero rows, K tails that are not multiples of 4 or 32 — per-row / per-column scales keep
# every row at the 3xTF32 accuracy relative to its own magnitude.
@pytest.mark.parametrize("tb", [False, True])
@pytest.mark.parametrize("shape", [(700, 256, 256), (300, 47, 101), (129, 256, 37), (64, 16, 3), (513, 100, 602)])
def test_gemm_f16_row_scales(shape, tb):
    m, n, k = shape
    rng = np.random.default_rng(m + n + k + tb)
    a = rng.uniform(-1, 1, (m, k)) * 10.0 ** rng.integers(-15, 15, (m, 1))
    a[::7] = 0.0
    b = rng.uniform(-1, 1, (n, k) if tb else (k, n))
    a, b = a.astype(np.float32), b.astype(np.float32)
    if tb:
        b *= (10.0 ** rng.integers(-10, 10, (n, 1))).astype(np.float32)
    else:
        b *= (10.0 ** rng.integers(-10, 10, (1, n))).astype(np.float32)
    ref = a.astype(np.float64) @ (b.astype(np.float64).T if tb else b.astype(np.float64))
    R.set_tuning("gemm_f16", 1)
    R.set_tuning("gemm_f16_min_k", 0)
    try:
        got = run_gemm(a, b, False, tb, mode=R.GEMM_TF32X3)
    finally:
        R.set_tuning("gemm_f16", 0)
        R.set_tuning("gemm_f16_min_k", 128)
    scale = np.abs(a).max(1, keepdims=True).astype(np.float64) * np.abs(b).max(1 if tb else 0)[None, :].astype(np.float64)
    err = np.abs(got - ref) / np.maximum(scale * k, 1e-300)
    assert np.all(np.isfinite(got)) and err.max() <= 1e-6, err.max()


@pytest.mark.parametrize("kernel", [1, 2, 3, 30])
def test_gemm_tcgen05_deterministic(gemm_kernel):
    rng = np.random.default_rng(5)
    a = rng.normal(size=(20000, 256)).astype(np.float32)
    b = rng.normal(size=(20000, 47)).astype(np.float32)
    r1 = run_gemm(a, b, True, False, mode=R.GEMM_TF32X3)
    r2 = run_gemm(a, b, True, False, mode=R.GEMM_TF32X3)
    assert bits_equal(r1, r2)


@pytest.mark.parametrize("knob,value", [("gemm3_cluster", 2), ("gemm3_wring", 64 << 10), ("gemm3_wring", 128 << 10)])
def test_gemm_v3_variants_bitwise(knob, value):
    """The v3 NN / NT pipeline variants (2-CTA W multicast, W-ring depth) reorder no arithmetic: every
    epilogue gives the default kernel's bits."""
    rng = np.random.default_rng(17)
    cases = [((777, 256), (256, 256), False), ((1000, 100), (100, 256), False), ((513, 47), (256, 47), True),
             ((300, 256), (48, 256), True)]
    base = []
    for (am, ak), bs, tb in cases:
        a = rng.uniform(-1, 1, (am, ak)).astype(np.float32)
        b = rng.uniform(-1, 1, bs).astype(np.float32)
        n = bs[0] if tb else bs[1]
        c0 = rng.normal(size=(am, n)).astype(np.float32)
        base.append((a, b, tb, c0, [run_gemm(a, b, False, tb, epi=e, c0=c0 if e == 1 else None, mode=R.GEMM_TF32X3)
                                    for e in (0, 1, 2)]))
    default = 96 << 10 if knob == "gemm3_wring" else 1
    R.set_tuning(knob, value)
    try:
        for a, b, tb, c0, outs in base:
            for e, ref in zip((0, 1, 2), outs):
                got = run_gemm(a, b, False, tb, epi=e, c0=c0 if e == 1 else None, mode=R.GEMM_TF32X3)
                assert bits_equal(got, ref), (knob, value, a.shape, tb, e)
    finally:
        R.set_tuning(knob, default)


# ---------------------------------------------------------------------------- MG_SPMM_FAST
# FMA and hub rows cut into fixed segments summed in order: deterministic, and as close to the exact
# (fp64) product as the reference's own serial fp32 sum is (normwise <= 1e-5 here, the model-level
# tolerance is 1e-4).
@pytest.mark.parametrize("w", [4, 48, 256, 300])
@pytest.mark.parametrize("seg", [64, 2048])
def test_spmm_fast_with_hubs(port32, port64, w, seg):
    from gpu_util import normwise
    rng = np.random.default_rng(11 + w + seg)
    rows, cols = 300, 5000
    rp, ci, v = random_tile(rng, rows, cols, 0.003, hub_rows=(0, 5, 299), hub_len=4800)
    h = rng.uniform(-1, 1, (cols, w)).astype(np.float32)
    o0 = rng.uniform(-1, 1, (rows, w)).astype(np.float32)
    ref = port32.spmm(rows, cols, rp, ci, v, h, True, o0)
    exact = port64.spmm(rows, cols, rp, ci, v.astype(np.float64), h.astype(np.float64), True, o0.astype(np.float64))
    R.set_tuning("heavy_row", 1000)
    R.set_tuning("fast_segment", seg)
    try:
        out = run_spmm(rp, ci, v, h, True, o0, mode=R.SPMM_FAST)
        out2 = run_spmm(rp, ci, v, h, True, o0, mode=R.SPMM_FAST)
        relu = run_spmm(rp, ci, v, h, True, o0, relu=True, mode=R.SPMM_FAST)
    finally:
        R.set_tuning("heavy_row", 4096)
        R.set_tuning("fast_segment", 2048)
    assert normwise(out, exact) <= 1e-5 and normwise(ref, exact) <= 1e-5
    assert bits_equal(out, out2)  # deterministic
    assert np.all(relu >= 0) and normwise(relu, np.maximum(exact, 0)) <= 1e-5
