"""Size-independent properties of the device kernels, restating the reference's unit tests
(tests/test_sparse.cpp:147-221, tests/test_dense.cpp:54-209, tests/test_gcn.cpp:243-253) for every
arithmetic mode the product ships — EXACT / FAST SpMM and EXACT / TF32X3 / TF32 GeMM."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
from gpu_util import bits_equal, dev_padded, normwise  # noqa: E402
from test_gpu_kernels import random_tile, run_gemm, run_spmm  # noqa: E402

from paper_2110_08688_b200 import rowgcn as R  # noqa: E402

SPMM_MODES = [R.SPMM_EXACT, R.SPMM_FAST]
GEMM_MODES = [R.GEMM_EXACT, R.GEMM_TF32X3, R.GEMM_TF32]


def csr(rows, edges):
    """CSR arrays from (row, col, val) triples sorted by (row, col)."""
    edges = sorted(edges)
    rp = np.zeros(rows + 1, np.int64)
    for r, _, _ in edges:
        rp[r + 1] += 1
    return np.cumsum(rp), np.array([c for _, c, _ in edges], np.int64), np.array([v for *_, v in edges], np.float32)


@pytest.mark.parametrize("mode", SPMM_MODES)
def test_spmm_identity_and_permutation(mode):
    rng = np.random.default_rng(33)
    h = rng.uniform(-1, 1, (4, 3)).astype(np.float32)
    rp, ci, v = csr(4, [(i, i, 1.0) for i in range(4)])
    assert bits_equal(run_spmm(rp, ci, v, h, mode=mode), h)
    rp, ci, v = csr(2, [(0, 1, 1.0), (1, 0, 1.0)])
    out = run_spmm(rp, ci, v, np.array([[1, 2], [3, 4]], np.float32), mode=mode)
    assert out.tolist() == [[3, 4], [1, 2]]


@pytest.mark.parametrize("mode", SPMM_MODES)
@pytest.mark.parametrize("w", [8, 48, 256])
def test_spmm_dense_oracle_linearity_accumulate(mode, w):
    rng = np.random.default_rng(45 + w)
    rows = cols = 400
    rp, ci, v = random_tile(rng, rows, cols, 0.05)
    dense = np.zeros((rows, cols))
    for r in range(rows):
        dense[r, ci[rp[r]:rp[r + 1]]] = v[rp[r]:rp[r + 1]]
    h1 = rng.uniform(-1, 1, (cols, w)).astype(np.float32)
    h2 = rng.uniform(-1, 1, (cols, w)).astype(np.float32)
    o1 = run_spmm(rp, ci, v, h1, mode=mode)
    assert normwise(o1, dense @ h1.astype(np.float64)) <= 1e-6
    o2 = run_spmm(rp, ci, v, h2, mode=mode)
    osum = run_spmm(rp, ci, v, h1 + h2, mode=mode)
    assert normwise(osum, o1.astype(np.float64) + o2) <= 1e-6
    assert bits_equal(run_spmm(rp, ci, v, 2 * h1, mode=mode), 2 * o1)  # power-of-two scaling is exact
    acc = run_spmm(rp, ci, v, h1, accumulate=True, out0=o1, mode=mode)
    assert normwise(acc, 2.0 * o1) <= 1e-6
    # row-parallel execution is deterministic (test_sparse.cpp:211-221)
    assert bits_equal(run_spmm(rp, ci, v, h1, mode=mode), o1)


@pytest.mark.parametrize("mode", SPMM_MODES)
def test_spmm_relu_forward_idempotent(mode):
    rng = np.random.default_rng(5)
    rp, ci, v = random_tile(rng, 64, 64, 0.1)
    h = rng.uniform(-1, 1, (64, 16)).astype(np.float32)
    plain = run_spmm(rp, ci, v, h, mode=mode)
    relu = run_spmm(rp, ci, v, h, relu=True, mode=mode)
    assert bits_equal(relu, np.maximum(plain, np.float32(0)))
    eye = csr(64, [(i, i, 1.0) for i in range(64)])
    assert bits_equal(run_spmm(*eye, relu, relu=True, mode=mode), relu)  # relu(relu(x)) == relu(x)


@pytest.mark.parametrize("mode", GEMM_MODES)
def test_gemm_identity_and_hand_arithmetic(mode):
    a = np.array([[1, 2], [3, 4]], np.float32)
    b = np.array([[5, 6], [7, 8]], np.float32)
    for ta, tb in ((False, False), (True, False), (False, True)):
        out = run_gemm(a.T.copy() if ta else a, b.T.copy() if tb else b, ta, tb, mode=mode)
        assert out.tolist() == [[19, 22], [43, 50]], (ta, tb)
    rng = np.random.default_rng(1)
    b = rng.uniform(-1, 1, (3, 2)).astype(np.float32)
    out = run_gemm(np.eye(3, dtype=np.float32), b, False, False, mode=mode)
    if mode == R.GEMM_EXACT:
        assert bits_equal(out, b)
    else:  # the TF32 split represents 22 of fp32's 24 significand bits (one term: 11)
        assert normwise(out, b) <= (1e-6 if mode == R.GEMM_TF32X3 else 1e-3)


@pytest.mark.parametrize("mode", GEMM_MODES)
def test_gemm_relu_epilogues(mode):
    """relu_backward mask (dense.hpp:221-231): out = act > 0 ? upstream : 0, out aliasing act (the step
    writes H_G straight into ahw[l-1]); relu_forward on the result (dense.hpp:208-215)."""
    up = np.array([[5.0, 5.0]], np.float32)
    act = np.array([[0.0, 3.0]], np.float32)
    out = run_gemm(up, np.eye(2, dtype=np.float32), False, False, epi=1, c0=act, mode=mode)
    assert out.tolist() == [[0.0, 5.0]]
    rng = np.random.default_rng(13)
    u = rng.uniform(-1, 1, (130, 40)).astype(np.float32)
    w = rng.uniform(-1, 1, (24, 40)).astype(np.float32)
    a_pos = rng.uniform(0.1, 1.0, (130, 24)).astype(np.float32)
    full = run_gemm(u, w, False, True, mode=mode)
    assert bits_equal(run_gemm(u, w, False, True, epi=1, c0=a_pos, mode=mode), full)  # positive act passes through
    act = rng.uniform(-1, 1, (130, 24)).astype(np.float32)
    assert bits_equal(run_gemm(u, w, False, True, epi=1, c0=act, mode=mode), np.where(act > 0, full, np.float32(0)))
    fwd = run_gemm(u, w, False, True, epi=2, mode=mode)
    assert bits_equal(fwd, np.maximum(full, np.float32(0)))


def test_adam_zero_gradient_leaves_w_unchanged():
    w = np.array([1.5, 0.0, 0.0, -2.5], np.float32)
    bufs = [dev_padded(x.reshape(1, 4)) for x in (w, np.zeros(4), np.zeros(4), np.zeros(4))]
    R.dev_adam(*[b.data_ptr() for b in bufs], 4, 1)
    torch.cuda.synchronize()
    assert bits_equal(bufs[0].cpu().numpy()[0], w)
