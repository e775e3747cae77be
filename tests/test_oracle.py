"""Pins the C restatement (oracle/oracle.c) against the reference's own golden vectors
(tests/golden/reference_golden.npz, made by tests/golden/make_golden.py from the compiled reference)
and, when oracle/_ref is built, against the reference directly. CPU only."""
import hashlib

import numpy as np
import pytest

from oracle.pyoracle import Dataset


def test_mt19937_64_known_answer(port32):
    # std::mt19937_64 with the default seed 5489: the 10000th output is standard-mandated
    # ([rand.predef]); inc/rng.hpp:9-12 relies on exactly this sequence.
    out = port32.rng_first(5489, 10000)
    assert int(out[-1]) == 9981545732273789042


def test_permutation_kats(port32, golden):
    # tests/test_partition.cpp:90-95
    assert list(port32.random_permutation(8, 7)[1]) == [2, 3, 5, 6, 1, 0, 4, 7]
    assert np.array_equal(port32.random_permutation(8, 7)[1], golden["perm_8_7_inverse"])
    fwd = port32.random_permutation(2708, 1)[0]
    assert list(fwd[:8]) == [1256, 858, 985, 2689, 2252, 1673, 2398, 1357]
    assert np.array_equal(fwd, golden["perm_2708_1_forward"])


@pytest.mark.parametrize("n,p", [(10, 4), (8, 8), (5, 8), (2449029, 8), (169343, 2), (232965, 4)])
def test_uniform_partition(port32, golden, n, p):
    assert np.array_equal(port32.uniform_partition(n, p), golden[f"partition_{n}_{p}"])
    if (n, p) == (10, 4):
        assert list(golden["partition_10_4"]) == [0, 2, 5, 7, 10]


def test_synth_graph_matches_reference(port32, golden):
    ds = port32.synth(300, 6.0, 0.7, 3, 12, 5)
    for k in ("row_ptr", "col_idx", "values", "features", "labels"):
        assert np.array_equal(getattr(ds, k), golden[f"synth300_{k}"]), k
    c1 = port32.synth(2708, 3.9, 0.7, 1, 1433, 7)
    assert c1.nnz == 10566
    assert np.array_equal(c1.row_ptr, golden["c1_row_ptr"])
    assert np.array_equal(c1.col_idx, golden["c1_col_idx"])
    assert np.array_equal(c1.labels, golden["c1_labels"])
    assert hashlib.sha256(c1.features.tobytes()).hexdigest() == golden["c1_features_sha256"].tobytes().decode()


def _small(golden):
    return Dataset(300, golden["synth300_row_ptr"], golden["synth300_col_idx"], golden["synth300_values"],
                   golden["synth300_features"], golden["synth300_labels"])


def test_prepare_tiles_bit_exact(port32, golden):
    prep = port32.prepare(_small(golden), permute=True, seed=9, workers=3)
    assert np.array_equal(prep.bounds, golden["prep300_bounds"])
    assert np.array_equal(prep.perm_forward, golden["prep300_perm"])
    assert np.array_equal(prep.features, golden["prep300_features"])
    for d in (0, 1):
        for i in range(3):
            for j in range(3):
                rp, ci, v = prep.tiles[d][i][j]
                assert np.array_equal(rp, golden[f"prep300_t{d}{i}{j}_rp"])
                assert np.array_equal(ci, golden[f"prep300_t{d}{i}{j}_ci"])
                assert np.array_equal(v, golden[f"prep300_t{d}{i}{j}_v"])


@pytest.mark.parametrize("k", range(4))
@pytest.mark.parametrize("s", ["f32", "f64"])
def test_spmm_bitwise(port32, port64, golden, k, s):
    port = port32 if s == "f32" else port64
    rp, ci, v = golden[f"spmm{k}_{s}_rp"], golden[f"spmm{k}_{s}_ci"], golden[f"spmm{k}_{s}_v"]
    h = golden[f"spmm{k}_{s}_h"]
    n = len(rp) - 1
    assert np.array_equal(port.spmm(n, n, rp, ci, v, h), golden[f"spmm{k}_{s}_out"])
    assert np.array_equal(port.spmm(n, n, rp, ci, v, h, True, golden[f"spmm{k}_{s}_o0"]), golden[f"spmm{k}_{s}_acc"])


@pytest.mark.parametrize("k,ta,tb", [(0, False, False), (1, True, False), (2, False, True), (3, True, True)])
@pytest.mark.parametrize("s", ["f32", "f64"])
def test_gemm_bitwise(port32, port64, golden, k, ta, tb, s):
    port = port32 if s == "f32" else port64
    out = port.gemm(golden[f"gemm{k}_{s}_a"], golden[f"gemm{k}_{s}_b"], ta, tb)
    assert np.array_equal(out, golden[f"gemm{k}_{s}_out"])


@pytest.mark.parametrize("s", ["f32", "f64"])
def test_softmax_xent_and_adam(port32, port64, golden, s):
    port = port32 if s == "f32" else port64
    m = golden[f"xent_{s}_mask"]
    ls, grad = port.softmax_xent_sum(golden[f"xent_{s}_logits"], golden[f"xent_{s}_labels"], m, int(m.sum()) + 3)
    assert ls == golden[f"xent_{s}_loss"][0]
    assert np.array_equal(grad, golden[f"xent_{s}_grad"])
    outs = port.adam(*(golden[f"adam_{s}_{nm}_in"] for nm in "wgmv"), 3, lr=0.05)
    for nm, arr in zip("wgmv", outs):
        assert np.array_equal(arr, golden[f"adam_{s}_{nm}_out"]), nm


@pytest.mark.parametrize("perm", [0, 1])
def test_c1_trajectory(port32, port64, golden, perm):
    """C1 Cora-shaped [1433,16,7], 5 epochs: f32 losses and W hashes bitwise, f64 losses bitwise."""
    from oracle.pyoracle import fnv1a
    ds = port32.synth(2708, 3.9, 0.7, 1, 1433, 7)
    m = port32.model(ds, [1433, 16, 7], 1, seed=1, permute=bool(perm))
    for e in range(5):
        assert m.step(e + 1)["loss"] == golden[f"c1_f32_perm{perm}_loss"][e]
        if e == 4:
            assert fnv1a(m.get_w()) == int(golden[f"c1_f32_perm{perm}_hash"][e])
    ds64 = port64.synth(2708, 3.9, 0.7, 1, 1433, 7)
    m64 = port64.model(ds64, [1433, 16, 7], 1, seed=1, permute=bool(perm))
    assert [m64.step(e + 1)["loss"] for e in range(5)] == list(golden[f"c1_f64_perm{perm}_loss"])


def test_c1_p_invariance(port32, golden):
    ds = port32.synth(2708, 3.9, 0.7, 1, 1433, 7)
    for P in (2, 4, 8):
        m = port32.model(ds, [1433, 16, 7], P, seed=1, permute=True)
        losses = [m.step(e + 1)["loss"] for e in range(5)]
        assert losses == list(golden[f"c1_f32_perm1_P{P}_loss"])
        assert np.array_equal(golden[f"c1_f32_perm1_P{P}_hash"], golden["c1_f32_perm1_hash"])  # ref's own claim


def test_step_dump(port32, golden):
    m = port32.model(_small(golden), [12, 8, 6, 5], 2, seed=5, permute=True)
    d = m.step(1, mode=0, dumps=True)
    assert d["loss"] == pytest.approx(golden["dump300_loss"][0], rel=0, abs=0)
    for l in range(3):
        assert np.array_equal(d["ahw_fwd"][l], golden[f"dump300_ahw_fwd{l}"])
        assert np.array_equal(d["ahw_bwd"][l], golden[f"dump300_ahw_bwd{l}"])
        assert np.array_equal(d["w_grad"][l], golden[f"dump300_wgrad{l}"])
        assert np.array_equal(m.get_w()[l], golden[f"dump300_wafter{l}"])
    assert np.array_equal(d["loss_grad"], golden["dump300_loss_grad"])


def test_port_equals_reference_directly(port32, ref):
    """When the compiled reference is present, cross-check a fresh random case end to end."""
    from oracle.pyoracle import make_cfg
    ds = ref.synth(500, 10.0, 0.6, 77, 9, 4)
    cfg = make_cfg([9, 7, 4], epochs=3, seed=4, permute=True, overlap=True)
    r = ref.train_run(ds, cfg, 4)
    m = port32.model(ds, [9, 7, 4], 4, seed=4, permute=True)
    assert [m.step(e + 1)["loss"] for e in range(3)] == list(r["loss"])
