"""GPU parity of the full training step through the C ABI against the CPU oracles.

Tolerances (stated per north_star): exact modes give BITWISE forward activations (the forward never
touches expf/logf); everything downstream of the loss uses CUDA expf/logf (<= 2 ulp vs glibc), so loss
is compared to the f64 reference at rel <= 1e-4 and per-layer gradient tensors to the f32 reference
with max|d| / max|ref| <= 1e-4. Multi-worker runs (P = 2, 4) use the in-process transport on one GPU.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
from gpu_util import bits_equal, normwise  # noqa: E402

from oracle.pyoracle import Dataset as ODs  # noqa: E402
from paper_2110_08688_b200 import rowgcn as R  # noqa: E402

TOL = 1e-4


def cfgx(*a, **k):
    """GcnConfig in the bitwise-parity modes unless a test asks for the tcgen05 / fast ones."""
    k.setdefault("gemm_mode", R.GEMM_EXACT)
    k.setdefault("spmm_mode", R.SPMM_EXACT)
    return R.GcnConfig(*a, **k)


def small_ds(golden):
    return (R.Dataset.from_arrays(golden["synth300_row_ptr"], golden["synth300_col_idx"], golden["synth300_values"],
                                  golden["synth300_features"], golden["synth300_labels"]),
            ODs(300, golden["synth300_row_ptr"], golden["synth300_col_idx"], golden["synth300_values"],
                golden["synth300_features"], golden["synth300_labels"]))


def group(ds, cfg, P):
    prep = R.prepare_data(ds, cfg, P)
    g = R.Group(cfg, prep, P, devices=[0] * P, transport=R.TRANSPORT_NCCL if P == 1 else R.TRANSPORT_LOCAL)
    g.init_params()
    return g


def gather(g, which, layer, P):
    return np.concatenate([g.read(which, layer, r) for r in range(P)], axis=0)


@pytest.mark.parametrize("P", [1, 2, 4])
@pytest.mark.parametrize("overlap", [False, True])
def test_forward_bitwise(golden, port32, P, overlap):
    ds, ods = small_ds(golden)
    cfg = cfgx([12, 8, 6, 5], seed=5, permute=True, overlap=overlap)
    m = port32.model(ods, [12, 8, 6, 5], P, seed=5, permute=True)
    ref = m.step(1, mode=2, dumps=True)["ahw_fwd"]
    with group(ds, cfg, P) as g:
        g.forward()
        for l in range(3):
            assert bits_equal(gather(g, R.T_AHW, l, P), ref[l]), f"layer {l}"


def test_step_dump_vs_reference(golden):
    """Teacher-forced train_step(1) on the small graph at P=2 vs the compiled reference's dump."""
    ds, _ = small_ds(golden)
    cfg = cfgx([12, 8, 6, 5], seed=5, permute=True, overlap=True)
    with group(ds, cfg, 2) as g:
        g.forward()
        for l in range(3):
            assert bits_equal(gather(g, R.T_AHW, l, 2), golden[f"dump300_ahw_fwd{l}"])
    with group(ds, cfg, 2) as g:
        g.compute_gradients()
        for l in range(3):
            assert normwise(g.read(R.T_WGRAD, l), golden[f"dump300_wgrad{l}"]) <= TOL
        for l in range(2):  # H-grads written into ahw[l] (relu-masked), gcn.hpp:345-347
            assert normwise(gather(g, R.T_AHW, l, 2), golden[f"dump300_ahw_bwd{l}"]) <= TOL
        assert normwise(gather(g, R.T_AHW, 2, 2), golden["dump300_loss_grad"]) <= TOL
    with group(ds, cfg, 2) as g:
        loss = g.train_step(1)
        assert abs(loss - golden["dump300_loss"][0]) <= TOL * abs(golden["dump300_loss"][0])
        for l in range(3):
            assert normwise(g.read(R.T_W, l), golden[f"dump300_wafter{l}"]) <= TOL
            assert np.all(g.read(R.T_WGRAD, l) == 0)  # grads zeroed after Adam (gcn.hpp:83)


@pytest.mark.parametrize("perm", [0, 1])
def test_c1_trajectory(golden, perm):
    """C1 Cora-shaped [1433,16,7], 5 epochs at P=1: losses vs the reference (f32 and f64 runs)."""
    ds = R.synth_graph(2708, 3.9, 0.7, 1, 1433, 7)
    cfg = cfgx([1433, 16, 7], epochs=5, seed=1, permute=bool(perm))
    art = R.train_run(ds, cfg, R.TrainOptions(workers=1, devices=[0]))
    ref32 = golden[f"c1_f32_perm{perm}_loss"]
    ref64 = golden[f"c1_f64_perm{perm}_loss"]
    for e in range(5):
        assert abs(art.epoch_loss[e] - ref64[e]) <= TOL * abs(ref64[e])
        assert abs(art.epoch_loss[e] - ref32[e]) <= TOL * abs(ref32[e])
    np.testing.assert_allclose(art.epoch_acc, golden[f"c1_f32_perm{perm}_acc"], atol=2.0 / 2708)


def test_p_invariance_bitwise():
    """W after every step is bitwise identical for P in {1,2,4} (tests/test_gcn.cpp:323-348)."""
    ds = R.synth_graph(2000, 8.0, 0.5, 44, 16, 4)
    cfg = cfgx([16, 16, 4], epochs=4, seed=17, permute=True, overlap=True)
    base = R.train_run(ds, cfg, R.TrainOptions(workers=1, devices=[0]))
    for P in (2, 4):
        dist = R.train_run(ds, cfg, R.TrainOptions(workers=P, devices=[0] * P, transport=R.TRANSPORT_LOCAL))
        for e in range(cfg.epochs):
            assert all(h == dist.w_hashes[e][0] for h in dist.w_hashes[e])
            assert dist.w_hashes[e][0] == base.w_hashes[e][0]
            assert abs(dist.epoch_loss[e] - base.epoch_loss[e]) <= 1e-10 * abs(base.epoch_loss[e])
        for a, b in zip(dist.final_w, base.final_w):
            assert bits_equal(a, b)


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_empty_parts_more_workers_than_vertices(mode):
    """tests/test_dist_spmm.cpp:123-131: P > n leaves some workers with no rows (empty tiles, empty
    broadcasts); the trajectory equals P = 1 (bitwise in the exact modes, P-invariant in the fast ones)."""
    ds = R.synth_graph(6, 2.0, 0.5, 3, 4, 2)
    kw = {} if mode == "exact" else dict(gemm_mode=R.GEMM_TF32X3, spmm_mode=R.SPMM_FAST)
    cfg = cfgx([4, 5, 2], epochs=3, seed=2, permute=True, overlap=True, **kw)
    base = R.train_run(ds, cfg, R.TrainOptions(workers=1, devices=[0]))
    dist = R.train_run(ds, cfg, R.TrainOptions(workers=8, devices=[0] * 8, transport=R.TRANSPORT_LOCAL))
    assert dist.epoch_loss == base.epoch_loss
    for a, b in zip(dist.final_w, base.final_w):
        assert bits_equal(a, b)


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_zero_upstream_and_backward_linearity(mode):
    """tests/test_gcn.cpp:227-241: a zero logits gradient gives zero W_G and zero H_G (ahw[0]); and the
    backward pass is linear in its upstream gradient — 2G gives exactly 2 W_G (power-of-two scaling)."""
    kw = {} if mode == "exact" else dict(gemm_mode=R.GEMM_TF32X3, spmm_mode=R.SPMM_FAST)
    dims = [4, 3, 2]
    ds = R.synth_graph(300, 5.0, 0.6, 47, dims[0], dims[-1])
    cfg = cfgx(dims, seed=3, permute=True, aggregate_input=False, **kw)
    P = 2
    with group(ds, cfg, P) as g:
        g.forward()
        for r in range(P):
            g.write(R.T_AHW, len(dims) - 2, np.zeros((g.rows(r)[1], dims[-1]), np.float32), r)
        g.backward()
        for l in range(len(dims) - 1):
            assert not g.read(R.T_WGRAD, l).any()
        for r in range(P):
            assert not g.read(R.T_AHW, 0, r).any()
        rng = np.random.default_rng(1)
        ups = [rng.normal(0, 1e-3, (g.rows(r)[1], dims[-1])).astype(np.float32) for r in range(P)]
        wg = []
        for scale in (1, 2):
            g.forward()
            for r in range(P):
                g.write(R.T_AHW, len(dims) - 2, scale * ups[r], r)
            g.backward()
            wg.append([g.read(R.T_WGRAD, l) for l in range(len(dims) - 1)])
        for a, b in zip(*wg):
            assert a.any() and bits_equal(b, 2 * a)


def test_overlap_on_equals_off():
    ds = R.synth_graph(600, 6.0, 0.6, 27, 4, 2)
    cfg = cfgx([4, 6, 2], epochs=3, seed=15)
    a = R.train_run(ds, cfg, R.TrainOptions(workers=4, devices=[0] * 4, transport=R.TRANSPORT_LOCAL))
    cfg.overlap = True
    b = R.train_run(ds, cfg, R.TrainOptions(workers=4, devices=[0] * 4, transport=R.TRANSPORT_LOCAL))
    assert a.epoch_loss == b.epoch_loss
    assert all(bits_equal(x, y) for x, y in zip(a.final_w, b.final_w))


def test_identity_pipeline_and_cycle():
    # tests/test_gcn.cpp:111-153: A = I, W = I passes the (nonnegative) features through
    n = 6
    rng = np.random.default_rng(5)
    x = rng.uniform(0, 1, (n, 3)).astype(np.float32)
    eye = R.Dataset.from_arrays(np.arange(n + 1), np.arange(n), np.ones(n, np.float32), x, np.zeros(n, np.int32))
    cfg = cfgx([3, 3, 3])
    with group(eye, cfg, 2) as g:
        g.set_params([np.eye(3, dtype=np.float32)] * 2)
        g.forward()
        assert np.array_equal(gather(g, R.T_AHW, 1, 2), x)
    cyc = R.Dataset.from_arrays([0, 1, 2], [1, 0], np.ones(2, np.float32), np.array([[1.0], [2.0]], np.float32),
                                np.zeros(2, np.int32))
    with group(cyc, cfgx([1, 1]), 1) as g:
        g.set_params([np.array([[3.0]], np.float32)])
        g.forward()
        assert list(g.read(R.T_AHW, 0).ravel()) == [6.0, 3.0]


def test_buffer_plan_and_no_step_allocations():
    ds = R.synth_graph(400, 6.0, 0.6, 71, 5, 3)
    for dims in ([5, 3], [5, 6, 3], [5, 6, 6, 3]):
        with group(ds, cfgx(dims, seed=3), 2) as g:
            lb, allocs0, _ = g.buffer_audit()
            assert lb == len(dims) - 1 + 3
            for t in (1, 2, 3):
                g.train_step(t)
            assert g.buffer_audit()[1] == allocs0 == 0


def test_label_out_of_range_raises():
    ds = R.Dataset.from_arrays([0, 1, 2], [1, 0], np.ones(2, np.float32), np.ones((2, 2), np.float32),
                               np.array([0, 5], np.int32))
    with group(ds, cfgx([2, 2]), 1) as g:
        with pytest.raises(R.ValueError, match="out of range"):
            g.train_step(1)


def test_loss_only_keeps_logits_and_matches_train_loss():
    ds = R.synth_graph(500, 6.0, 0.6, 3, 8, 4)
    cfg = cfgx([8, 8, 4], seed=2, permute=True)
    with group(ds, cfg, 2) as g:
        l0 = g.loss_only()
        logits = gather(g, R.T_AHW, 1, 2)
        g.forward()
        assert bits_equal(gather(g, R.T_AHW, 1, 2), logits)
        l1 = g.compute_gradients()
        assert abs(l0 - l1) <= 1e-12 * abs(l1)


@pytest.mark.parametrize("mode,tol", [(R.GEMM_TF32X3, 1e-4)])
def test_step_dump_tcgen05(golden, mode, tol):
    """The same teacher-forced step with the tcgen05 GeMMs: every tensor within the stated tolerance."""
    ds, _ = small_ds(golden)
    cfg = cfgx([12, 8, 6, 5], seed=5, permute=True, overlap=True, gemm_mode=mode)
    with group(ds, cfg, 2) as g:
        g.forward()
        for l in range(3):
            assert normwise(gather(g, R.T_AHW, l, 2), golden[f"dump300_ahw_fwd{l}"]) <= 1e-5
    with group(ds, cfg, 2) as g:
        g.compute_gradients()
        for l in range(3):
            assert normwise(g.read(R.T_WGRAD, l), golden[f"dump300_wgrad{l}"]) <= tol
        for l in range(2):
            assert normwise(gather(g, R.T_AHW, l, 2), golden[f"dump300_ahw_bwd{l}"]) <= tol
    with group(ds, cfg, 2) as g:
        loss = g.train_step(1)
        assert abs(loss - golden["dump300_loss"][0]) <= tol * abs(golden["dump300_loss"][0])
        for l in range(3):
            assert normwise(g.read(R.T_W, l), golden[f"dump300_wafter{l}"]) <= tol


def test_c1_trajectory_tcgen05(golden):
    ds = R.synth_graph(2708, 3.9, 0.7, 1, 1433, 7)
    cfg = cfgx([1433, 16, 7], epochs=5, seed=1, permute=True, gemm_mode=R.GEMM_TF32X3)
    art = R.train_run(ds, cfg, R.TrainOptions(workers=1, devices=[0]))
    ref64 = golden["c1_f64_perm1_loss"]
    for e in range(5):
        assert abs(art.epoch_loss[e] - ref64[e]) <= TOL * abs(ref64[e])


def test_p_invariance_bitwise_tcgen05():
    """The tcgen05 path is deterministic and row-local, and the W-grad split-K chunks are fixed relative to the
    canonical blocks, so the W trajectory stays bitwise P-invariant in TF32X3 mode too."""
    ds = R.synth_graph(9000, 8.0, 0.5, 44, 16, 4)
    cfg = cfgx([16, 32, 4], epochs=3, seed=17, permute=True, overlap=True, gemm_mode=R.GEMM_TF32X3)
    base = R.train_run(ds, cfg, R.TrainOptions(workers=1, devices=[0]))
    for P in (2, 4):
        dist = R.train_run(ds, cfg, R.TrainOptions(workers=P, devices=[0] * P, transport=R.TRANSPORT_LOCAL))
        for e in range(cfg.epochs):
            assert all(h == dist.w_hashes[e][0] for h in dist.w_hashes[e])
            assert dist.w_hashes[e][0] == base.w_hashes[e][0]


def test_fast_modes_trajectory_and_determinism(golden):
    """TF32X3 GeMMs + fast SpMM (the benchmark configuration): C1 losses within 1e-4 of the f64 reference,
    run-to-run bitwise deterministic, and W bitwise P-invariant when no row is split (P-invariance with
    hub segments holds up to the segment boundaries, which depend on the tile)."""
    ds = R.synth_graph(2708, 3.9, 0.7, 1, 1433, 7)
    cfg = cfgx([1433, 16, 7], epochs=5, seed=1, permute=True, gemm_mode=R.GEMM_TF32X3,
                      spmm_mode=R.SPMM_FAST)
    a = R.train_run(ds, cfg, R.TrainOptions(workers=1, devices=[0]))
    b = R.train_run(ds, cfg, R.TrainOptions(workers=1, devices=[0]))
    ref64 = golden["c1_f64_perm1_loss"]
    for e in range(5):
        assert abs(a.epoch_loss[e] - ref64[e]) <= TOL * abs(ref64[e])
    assert a.epoch_loss == b.epoch_loss and a.w_hashes == b.w_hashes
    d = R.train_run(ds, cfg, R.TrainOptions(workers=2, devices=[0, 0], transport=R.TRANSPORT_LOCAL))
    for e in range(5):
        assert abs(d.epoch_loss[e] - a.epoch_loss[e]) <= 1e-6 * abs(a.epoch_loss[e])


def test_step_dump_fast_spmm(golden):
    ds, _ = small_ds(golden)
    cfg = cfgx([12, 8, 6, 5], seed=5, permute=True, overlap=True, gemm_mode=R.GEMM_TF32X3,
                      spmm_mode=R.SPMM_FAST)
    R.set_tuning("heavy_row", 8)  # force hub segments on this small graph
    R.set_tuning("fast_segment", 32)
    try:
        with group(ds, cfg, 2) as g:
            g.compute_gradients()
            for l in range(3):
                assert normwise(g.read(R.T_WGRAD, l), golden[f"dump300_wgrad{l}"]) <= TOL
            for l in range(2):
                assert normwise(gather(g, R.T_AHW, l, 2), golden[f"dump300_ahw_bwd{l}"]) <= TOL
    finally:
        R.set_tuning("heavy_row", 4096)
        R.set_tuning("fast_segment", 2048)


@pytest.mark.parametrize("P", [1, 3])
def test_aggregate_input_trajectory(ref, P):
    """aggregate_input (FAST default): layer 0 as (Â·X)·W0 with Â·X reused for W0's gradient. Same math as
    the reference's A·(X·W0) / X^T·(Â^T·G0); losses within 1e-4 of the f64 reference, final W within 1e-4
    of the f32 reference, and one extra n x d0 buffer in the plan."""
    from oracle.pyoracle import make_cfg
    dims = [20, 48, 24, 5]
    ds = R.synth_graph(3000, 8.0, 0.7, 11, dims[0], dims[-1])
    cfg = cfgx(dims, epochs=4, seed=2, permute=True, overlap=P > 1, gemm_mode=R.GEMM_TF32X3,
               spmm_mode=R.SPMM_FAST)
    assert cfg.aggregate_input
    got = R.train_run(ds, cfg, R.TrainOptions(workers=P, devices=[0] * P,
                                             transport=R.TRANSPORT_NCCL if P == 1 else R.TRANSPORT_LOCAL))
    rcfg = make_cfg(dims, epochs=4, seed=2, permute=True, overlap=P > 1)
    r64 = ref.train_run(ref.synth(3000, 8.0, 0.7, 11, dims[0], dims[-1], dtype=np.float64), rcfg, P, np.float64)
    r32 = ref.train_run(ref.synth(3000, 8.0, 0.7, 11, dims[0], dims[-1]), rcfg, P)
    for e in range(4):
        assert abs(got.epoch_loss[e] - r64["loss"][e]) <= TOL * abs(r64["loss"][e])
    for l in range(3):
        assert normwise(got.final_w[l], r32["final_w"][l]) <= TOL
    with group(ds, cfg, P) as g:
        assert g.buffer_audit()[0] == 3 + 3 + 1


def test_aggregate_input_ignored_in_exact_mode():
    ds = R.synth_graph(800, 6.0, 0.6, 4, 6, 3)
    a = R.train_run(ds, cfgx([6, 16, 3], epochs=2, seed=1, aggregate_input=True), R.TrainOptions(devices=[0]))
    b = R.train_run(ds, cfgx([6, 16, 3], epochs=2, seed=1, aggregate_input=False), R.TrainOptions(devices=[0]))
    assert a.epoch_loss == b.epoch_loss and a.w_hashes == b.w_hashes
