"""Kernel-level parity of the fused loss and optimizer kernels through the C ABI (mg_dev_softmax_xent,
mg_dev_adam), restating the reference's own unit tests on the GPU:
  * softmax_xent (tests/test_dense.cpp:211-297): ln C for uniform logits, saturated logit, unmasked rows
    exactly zero and masked rows summing to zero, shift invariance, the error contracts, and products-
    shaped rows against the compiled reference (f32 gradient, f64 loss);
  * argmax ties (inc/gcn.hpp:279-282: the first maximum wins);
  * adam_step (tests/test_gcn.cpp:255-285): the scalar first step is -lr, the two-step scalar oracle,
    t < 1 rejected — and bitwise equality with the compiled reference's f32 adam_step."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2110_08688_b200 import rowgcn as R  # noqa: E402


def dev(a, dtype=None):
    return torch.from_numpy(np.ascontiguousarray(a if dtype is None else a.astype(dtype))).cuda()


def run_softmax(logits, labels, mask, denom, ld=None):
    rows, c = logits.shape
    ld = ld or c
    buf = np.zeros((rows, ld), np.float32)
    buf[:, :c] = logits
    buf[:, c:] = 7.0  # padding must come back zeroed
    z = dev(buf)
    lab = dev(np.asarray(labels, np.int32))
    msk = dev(np.asarray(mask, np.uint8))
    loss, corr = R.dev_softmax_xent(z.data_ptr(), rows, c, ld, lab.data_ptr(), msk.data_ptr(), denom)
    torch.cuda.synchronize()
    g = z.cpu().numpy()
    assert not g[:, c:].any()
    return loss, corr, g[:, :c]


def test_uniform_logits_give_ln_c():
    loss, corr, _ = run_softmax(np.zeros((3, 4), np.float32), [0, 1, 3], [1, 1, 1], 3)
    assert abs(loss / 3 - math.log(4.0)) <= 1e-6
    assert corr == 1  # all ties: argmax = class 0, only row 0 is labelled 0


def test_saturated_true_logit():
    x = np.zeros((1, 3), np.float32)
    x[0, 1] = 1000.0
    loss, corr, g = run_softmax(x, [1], [1], 1)
    assert 0.0 <= loss < 1e-6 and corr == 1
    assert np.abs(g).max() < 1e-6


def test_gradient_properties_vs_reference(ref):
    rng = np.random.default_rng(23)
    n, c = 6, 5
    x = rng.uniform(-2, 2, (n, c)).astype(np.float32)
    labels = rng.integers(0, c, n).astype(np.int32)
    mask = np.array([1, 0, 1, 1, 0, 1], np.uint8)
    loss, _, g = run_softmax(x, labels, mask, int(mask.sum()))
    for i in range(n):
        if not mask[i]:
            assert not g[i].any()
        else:
            assert abs(float(g[i].astype(np.float64).sum())) < 1e-6
    l64, g64 = ref.softmax_xent_sum(x.astype(np.float64), labels, mask, int(mask.sum()))
    assert abs(loss - l64) <= 1e-6 * abs(l64)
    assert np.abs(g - g64).max() <= 1e-6 * np.abs(g64).max()


def test_shift_invariance():
    rng = np.random.default_rng(29)
    x = rng.uniform(-1, 1, (5, 4)).astype(np.float32)
    labels, mask = [0, 1, 2, 3, 0], [1] * 5
    base, _, _ = run_softmax(x, labels, mask, 5)
    x[2] += 37.5
    shifted, _, _ = run_softmax(x, labels, mask, 5)
    assert abs(base - shifted) < 1e-5


def test_error_contracts():
    x = np.zeros((2, 3), np.float32)
    with pytest.raises(R.ValueError, match="empty mask"):
        run_softmax(x, [0, 5], [0, 0], 0)
    with pytest.raises(R.ValueError, match="label 5 out of range"):
        run_softmax(x, [0, 5], [1, 1], 2)
    run_softmax(x, [0, 5], [1, 0], 1)  # unmasked rows are not checked (dense.hpp:255-262)


def test_argmax_first_max_wins():
    x = np.array([[1, 3, 3, 0], [2, 2, 2, 2], [0, 0, 5, 5], [4, 1, 4, 1]], np.float32)
    _, corr, _ = run_softmax(x, [1, 0, 2, 0], [1] * 4, 4)
    assert corr == 4
    _, corr, _ = run_softmax(x, [2, 1, 3, 2], [1] * 4, 4)
    assert corr == 0


@pytest.mark.parametrize("c,ld", [(47, 48), (7, 8), (40, 40), (172, 176), (256, 256)])
def test_products_rows_vs_reference(ref, c, ld):
    """Products-shaped logits (and the other configs' class counts) against the compiled reference."""
    rng = np.random.default_rng(c)
    n = 20000
    x = rng.normal(0, 3, (n, c)).astype(np.float32)
    labels = rng.integers(0, c, n).astype(np.int32)
    mask = (rng.random(n) < 0.8).astype(np.uint8)
    denom = 2449029  # the global masked count of a multi-GPU run, not this slice's
    loss, corr, g = run_softmax(x, labels, mask, denom, ld)
    l32, g32 = ref.softmax_xent_sum(x, labels, mask, denom)
    l64, _ = ref.softmax_xent_sum(x.astype(np.float64), labels, mask, denom)
    assert abs(loss - l64) <= 1e-6 * abs(l64)  # fp64 accumulation: closer to f64 than the reference's f32 sum
    # Σexp in warp-tree order vs the reference's serial order: a few ulps of the row sum
    assert np.abs(g - g32).max() <= 5e-6 * np.abs(g32).max()
    ok = mask.astype(bool)
    assert corr == int((np.argmax(x, axis=1) == labels)[ok].sum())


def run_adam(w, g, m, v, t, **kw):
    bufs = [dev(a, np.float32) for a in (w, g, m, v)]
    R.dev_adam(*[b.data_ptr() for b in bufs], w.size, t, **kw)
    torch.cuda.synchronize()
    return [b.cpu().numpy() for b in bufs]


def test_adam_scalar_first_step_and_two_step_oracle():
    z = np.zeros(1, np.float32)
    w, g, m, v = run_adam(z, np.ones(1, np.float32), z, z, 1, lr=0.1)
    assert abs(float(w[0]) + 0.1) < 1e-7 and g[0] == 0.0
    wo, mo, vo = 0.0, 0.0, 0.0
    for t in (1, 2):
        mo = 0.9 * mo + 0.1
        vo = 0.999 * vo + 0.001
        wo -= 0.1 * (mo / (1 - 0.9 ** t)) / (math.sqrt(vo / (1 - 0.999 ** t)) + 1e-8)
    w, m, v = z, z, z
    for t in (1, 2):
        w, _, m, v = run_adam(w, np.ones(1, np.float32), m, v, t, lr=0.1)
    assert abs(float(w[0]) - wo) < 1e-5  # f32 constants (1 - 0.999f is 1.3e-5 off 0.001) vs the double oracle
    with pytest.raises(R.ValueError, match="step index must be >= 1"):
        run_adam(w, np.ones(1, np.float32), m, v, 0)


@pytest.mark.parametrize("t", [1, 2, 7, 1000])
def test_adam_bitwise_vs_reference(ref, t):
    rng = np.random.default_rng(t)
    n = 256 * 47 + 5
    w = rng.normal(0, 0.1, n).astype(np.float32)
    g = rng.normal(0, 1e-3, n).astype(np.float32)
    m = rng.normal(0, 1e-4, n).astype(np.float32)
    v = rng.uniform(0, 1e-6, n).astype(np.float32)
    got = run_adam(w, g, m, v, t, lr=0.01)
    want = ref.adam(w, g, m, v, t, lr=0.01)
    for a, b in zip(got, want):
        assert a.tobytes() == b.tobytes()


def test_golden_vectors(golden):
    """The committed reference outputs (tests/golden/make_golden.py): softmax with denom = |mask| + 3 and
    Adam at t = 3, lr = 0.05 — the gradient within libm-vs-CUDA expf, the Adam update bitwise."""
    x, lab, msk = golden["xent_f32_logits"], golden["xent_f32_labels"], golden["xent_f32_mask"]
    denom = int(msk.sum()) + 3
    loss, _, g = run_softmax(x, lab, msk, denom)
    assert abs(loss - float(golden["xent_f32_loss"][0])) <= 1e-5 * abs(loss)
    ref_g = golden["xent_f32_grad"]
    assert np.abs(g - ref_g).max() <= 2e-6 * np.abs(ref_g).max()
    ins = [golden[f"adam_f32_{k}_in"] for k in "wgmv"]
    outs = run_adam(*ins, 3, lr=0.05)
    for k, a in zip("wgmv", outs):
        assert a.tobytes() == golden[f"adam_f32_{k}_out"].tobytes(), k
