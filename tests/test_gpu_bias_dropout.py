"""The default-off bias + dropout extension (mggcn.h mg_config.bias / .dropout; the reference has
neither, so there is no parity claim) against a float64 numpy restatement of the same model:

  z_l = Â^T-aggregate(H_l W_l) + b_l;  H_{l+1} = drop(relu(z_l)) for hidden layers (keep with prob 1 - p,
  scale 1 / (1 - p), mask = counter hash of (seed, step, layer, global row, column), mg_epi.cuh)

forward activations, masked softmax-CE loss, W_G and b_G (canonical-block sums), in the exact and in the
production arithmetic modes, P = 1 and 2 (in-process transport), plus bitwise P-invariance of W_G / b_G."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from gpu_util import normwise  # noqa: E402

from paper_2110_08688_b200 import rowgcn as R  # noqa: E402

M64 = (1 << 64) - 1


def mix64(z):
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def keep_mask(seed, t, layer, n, d, p):
    """mg_epi.cuh dropout_hash restated (Python integers, exact 64-bit wrap-around)."""
    key = mix64(seed ^ mix64(t * 1024 + layer + 1))
    thr = min(2 ** 32 - 1, int(np.floor(p * 2 ** 32)))
    out = np.zeros((n, d), bool)
    for r in range(n):
        for c in range(d):
            out[r, c] = (mix64((key + (r * 65536 + c) * 0x9E3779B97F4A7C15) & M64) >> 32) >= thr
    return out


def dense(prep, direction, n):
    P = prep.workers
    a = np.zeros((n, n))
    for i in range(P):
        for j in range(P):
            rp, ci, v = prep.tile(direction, i, j)
            r0, c0 = prep.bounds[i], prep.bounds[j]
            for u in range(len(rp) - 1):
                a[r0 + u, c0 + ci[rp[u]:rp[u + 1]]] = v[rp[u]:rp[u + 1]]
    return a


def restate(prep, dims, ws, bs, seed, p, t=1):
    """float64 forward + loss + backward of the step on the permuted rows."""
    n = prep.n
    x, lab, mask, _ = prep.rows_export(dims[0])
    F, B = dense(prep, 0, n), dense(prep, 1, n)
    L = len(dims) - 1
    h, acts, zs = x.astype(np.float64), [], []
    for l in range(L):
        z = F @ (h @ ws[l]) + bs[l]
        if l < L - 1:
            a = np.maximum(z, 0.0)
            if p > 0:
                a = np.where(keep_mask(seed, t, l, n, dims[l + 1], p), a / (1 - p), 0.0)
        else:
            a = z
        acts.append(a)
        h = a
    logits = acts[-1]
    e = np.exp(logits - logits.max(1, keepdims=True))
    sm = e / e.sum(1, keepdims=True)
    N = int(mask.sum())
    loss = float(-np.log(sm[np.arange(n), lab]).sum() / N)
    g = (sm - np.eye(dims[-1])[lab]) / N
    wg, bg = [None] * L, [None] * L
    for l in range(L - 1, -1, -1):
        h_in = x.astype(np.float64) if l == 0 else acts[l - 1]
        bg[l] = g.sum(0)
        hwg = B @ g
        wg[l] = h_in.T @ hwg
        if l > 0:
            g = (hwg @ ws[l].T) * (acts[l - 1] > 0) * (1.0 / (1 - p))
    return acts, loss, wg, bg


MODES = {"exact": dict(gemm_mode=R.GEMM_EXACT, spmm_mode=R.SPMM_EXACT),
         "production": dict(gemm_mode=R.GEMM_TF32X3, spmm_mode=R.SPMM_FAST, aggregate_input=True)}


@pytest.mark.parametrize("mode", ["exact", "production"])
@pytest.mark.parametrize("P", [1, 2])
@pytest.mark.parametrize("p", [0.0, 0.3])
def test_bias_dropout_step_vs_numpy(mode, P, p):
    dims = [6, 16, 8, 3]
    ds = R.synth_graph(300, 6.0, 0.6, 19, dims[0], dims[-1])
    cfg = R.GcnConfig(dims, seed=9, permute=True, overlap=P > 1, bias=True, dropout=p, **MODES[mode])
    prep = R.prepare_data(ds, cfg, P)
    rng = np.random.default_rng(3)
    bs = [rng.normal(0, 0.2, (1, dims[l + 1])).astype(np.float32) for l in range(len(dims) - 1)]
    tr = R.TRANSPORT_NCCL if P == 1 else R.TRANSPORT_LOCAL
    with R.Group(cfg, prep, P, devices=[0] * P, transport=tr) as g:
        g.init_params()
        for l, b in enumerate(bs):
            g.write(R.T_BIAS, l, b)
        ws = g.params()
        acts, loss, wg, bg = restate(prep, dims, [w.astype(np.float64) for w in ws], [b.astype(np.float64) for b in bs],
                                     9, p)
        got = g.compute_gradients()  # training pass of step 1: dropout active
        tol = 1e-5 if mode == "exact" else 1e-4
        assert abs(got - loss) <= tol * abs(loss)
        for l in range(len(dims) - 1):
            assert normwise(g.read(R.T_WGRAD, l), wg[l]) <= tol, l
            assert normwise(g.read(R.T_BIAS_GRAD, l), bg[l][None, :]) <= tol, l
        g.forward()  # evaluation forward: bias, no dropout
        ev, _, _, _ = restate(prep, dims, [w.astype(np.float64) for w in ws], [b.astype(np.float64) for b in bs], 9, 0.0)
        for l in range(len(dims) - 1):
            got_a = np.concatenate([g.read(R.T_AHW, l, r) for r in range(P)], axis=0)
            assert normwise(got_a, ev[l]) <= tol, l
    if p > 0:  # the mask is what the hash says, and about p of the hidden outputs are dropped
        m = keep_mask(9, 1, 0, 300, dims[1], p)
        assert abs(1 - m.mean() - p) < 0.05


def test_bias_gradients_p_invariant_and_adam():
    dims = [5, 12, 4]
    ds = R.synth_graph(800, 8.0, 0.6, 23, dims[0], dims[-1])
    runs = []
    for P in (1, 2, 4):
        cfg = R.GcnConfig(dims, epochs=3, seed=4, permute=True, overlap=True, bias=True, dropout=0.25)
        with R.Group(cfg, R.prepare_data(ds, cfg, P), P, devices=[0] * P,
                     transport=R.TRANSPORT_NCCL if P == 1 else R.TRANSPORT_LOCAL) as g:
            g.init_params()
            for t in (1, 2, 3):
                g.train_step(t)
            runs.append([g.read(R.T_W, l) for l in range(2)] + [g.read(R.T_BIAS, l) for l in range(2)])
    for other in runs[1:]:
        for a, b in zip(runs[0], other):
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert np.abs(runs[0][2]).max() > 0  # the biases moved (Adam updates them)


def test_bias_off_has_no_bias_tensor():
    ds = R.synth_graph(100, 4.0, 0.6, 1, 4, 2)
    cfg = R.GcnConfig([4, 4, 2], seed=1)
    with R.Group(cfg, R.prepare_data(ds, cfg, 1), 1, devices=[0]) as g:
        with pytest.raises(R.ValueError, match="no bias"):
            g.read(R.T_BIAS, 0)
    with pytest.raises(R.ConfigError, match="dropout"):
        R.GcnConfig([4, 4, 2], dropout=1.0).validate()
