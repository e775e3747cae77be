"""grad_run, the paper's optional schedule flags and end-to-end learning, against the compiled reference:
  * grad_run (inc/driver.hpp:216-251): W_G and loss of one forward/backward, every arithmetic mode, P = 1, 2;
  * order_swap (inc/gcn.hpp:145-148, :254-260) and skip_first_backward_spmm (:298-307) trajectories —
    the reference's test_gcn.cpp:155-190 / :395-415 cases;
  * central finite differences of the full model (tests/test_gcn.cpp:177-211, acceptance c2), in f32;
  * acceptance c9 (tests/acceptance.cpp:347-386): >= 95% accuracy on a 2-block community graph."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
from gpu_util import normwise  # noqa: E402

from paper_2110_08688_b200 import rowgcn as R  # noqa: E402

TOL = 1e-4
MODES = {"exact": (R.GEMM_EXACT, R.SPMM_EXACT), "tf32x3": (R.GEMM_TF32X3, R.SPMM_EXACT),
         "fast": (R.GEMM_TF32X3, R.SPMM_FAST)}


def opts(P):
    return dict(devices=[0] * P, transport=R.TRANSPORT_NCCL if P == 1 else R.TRANSPORT_LOCAL)


@pytest.mark.parametrize("P", [1, 2])
@pytest.mark.parametrize("mode", sorted(MODES))
def test_grad_run_vs_reference(ref, P, mode):
    from oracle.pyoracle import make_cfg
    gm, sm = MODES[mode]
    dims = [12, 24, 16, 5]
    ds = R.synth_graph(4000, 9.0, 0.7, 21, dims[0], dims[-1])
    got = R.grad_run(ds, R.GcnConfig(dims, seed=5, permute=True, gemm_mode=gm, spmm_mode=sm, aggregate_input=False),
                     P, **opts(P))
    r64 = ref.grad_run(ref.synth(4000, 9.0, 0.7, 21, dims[0], dims[-1], dtype=np.float64),
                       make_cfg(dims, seed=5, permute=True), P, np.float64)
    assert abs(got.loss - r64["loss"]) <= TOL * abs(r64["loss"])
    for l in range(len(dims) - 1):
        assert normwise(got.w_grad[l], r64["w_grad"][l]) <= TOL, l
    # the canonical 8-block W-grad reduction makes W_G independent of P (gcn.hpp:316-335)
    assert len(set(got.grad_hash_per_rank)) == 1


@pytest.mark.parametrize("flag", ["order_swap", "skip_first_backward_spmm"])
@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_schedule_flags_vs_reference(ref, flag, mode):
    """Each flag against the reference run with the same flag (trajectory + final W)."""
    from oracle.pyoracle import make_cfg
    gm, sm = MODES[mode]
    dims = [8, 32, 32, 4]  # d0 < d1: order_swap reorders layer 0
    ds = R.synth_graph(3000, 8.0, 0.7, 13, dims[0], dims[-1])
    kw = {flag: True}
    got = R.train_run(ds, R.GcnConfig(dims, epochs=4, seed=3, permute=True, overlap=True, gemm_mode=gm, spmm_mode=sm,
                                      aggregate_input=False, **kw), R.TrainOptions(workers=2, **opts(2)))
    rcfg = make_cfg(dims, epochs=4, seed=3, permute=True, overlap=True, **kw)
    r64 = ref.train_run(ref.synth(3000, 8.0, 0.7, 13, dims[0], dims[-1], dtype=np.float64), rcfg, 2, np.float64)
    r32 = ref.train_run(ref.synth(3000, 8.0, 0.7, 13, dims[0], dims[-1]), rcfg, 2)
    for e in range(4):
        assert abs(got.epoch_loss[e] - r64["loss"][e]) <= TOL * abs(r64["loss"][e])
    for l in range(len(dims) - 1):
        assert normwise(got.final_w[l], r32["final_w"][l]) <= TOL


def test_order_swap_changes_schedule_not_results():
    """tests/test_gcn.cpp:155-190: swapped and plain order agree (here in fp32 exact mode: the float
    association differs, so within rounding rather than bitwise)."""
    dims = [6, 20, 3]
    ds = R.synth_graph(2500, 7.0, 0.6, 3, dims[0], dims[-1])
    base = dict(epochs=3, seed=9, permute=True, gemm_mode=R.GEMM_EXACT, spmm_mode=R.SPMM_EXACT)
    a = R.train_run(ds, R.GcnConfig(dims, **base), R.TrainOptions(devices=[0]))
    b = R.train_run(ds, R.GcnConfig(dims, order_swap=True, **base), R.TrainOptions(devices=[0]))
    for x, y in zip(a.epoch_loss, b.epoch_loss):
        assert abs(x - y) <= 1e-5 * abs(x)


def test_finite_differences():
    """Central differences of the loss in W against the analytic W_G (f32, exact modes, h = 1e-2)."""
    dims = [5, 8, 3]
    ds = R.synth_graph(600, 6.0, 0.6, 8, dims[0], dims[-1])
    cfg = R.GcnConfig(dims, seed=4, permute=True, gemm_mode=R.GEMM_EXACT, spmm_mode=R.SPMM_EXACT)
    prep = R.prepare_data(ds, cfg, 1)
    rng = np.random.default_rng(0)
    with R.Group(cfg, prep, 1, devices=[0]) as g:
        g.init_params()
        w0 = [w.astype(np.float64) for w in g.params()]
        g.compute_gradients()
        grads = g.w_grads()
        checked = 0
        for l in range(len(dims) - 1):
            for _ in range(6):
                i, j = rng.integers(0, w0[l].shape[0]), rng.integers(0, w0[l].shape[1])
                if abs(grads[l][i, j]) < 1e-3:
                    continue
                vals = []
                for sgn in (1, -1):
                    ws = [w.copy() for w in w0]
                    ws[l][i, j] += sgn * 1e-2
                    g.set_params([w.astype(np.float32) for w in ws])
                    vals.append(g.loss_only())
                fd = (vals[0] - vals[1]) / 2e-2
                assert abs(fd - grads[l][i, j]) <= 2e-2 * abs(grads[l][i, j]) + 2e-4, (l, i, j, fd, grads[l][i, j])
                checked += 1
        assert checked >= 6


def two_block(seed=5150, n=1000):
    """acceptance.cpp:347-370 restated with numpy's RNG: 6 stubs per vertex, 90% inside its half."""
    rng = np.random.default_rng(seed)
    half = n // 2
    edges = set()
    for u in range(n):
        for _ in range(6):
            same = rng.random() < 0.9
            lo = 0 if (u < half) == same else half
            v = lo + int(rng.integers(0, half))
            if v != u:
                edges.add((u, v))
                edges.add((v, u))
    edges = sorted(edges)
    rp = np.zeros(n + 1, np.int64)
    for u, _ in edges:
        rp[u + 1] += 1
    rp = np.cumsum(rp)
    ci = np.array([v for _, v in edges], np.int64)
    labels = (np.arange(n) >= half).astype(np.int32)
    x = np.zeros((n, 4), np.float32)
    x[np.arange(n), labels] = 1.0
    x += (0.3 * rng.uniform(-1, 1, (n, 4))).astype(np.float32)
    return R.Dataset.from_arrays(rp, ci, np.ones(len(ci), np.float32), x, labels)


def test_c9_two_block_convergence():
    ds = two_block()
    art = R.train_run(ds, R.GcnConfig([4, 16, 2], epochs=200, seed=7, lr=0.01),
                      R.TrainOptions(workers=2, **opts(2)))
    assert max(art.epoch_acc) >= 0.95
    assert art.epoch_loss[-1] < art.epoch_loss[0]
