"""CPU tests of the C-ABI library's host half: it loads without a GPU, exports every symbol declared in
include/mggcn.h, and its generator + partitioner are bit-identical to the reference (via the pinned C
restatement and the golden fixtures). No device compute here."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2110_08688_b200 import rowgcn as R
from paper_2110_08688_b200._lib import LIB_PATH, SIGNATURES

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "mggcn.h")).read()
    return set(re.findall(r"^\s*(?:mg_status|void|const char\*|int32_t)\s+(mg_\w+)\s*\(", txt, re.M))


def test_library_exports_every_header_symbol():
    syms = header_symbols()
    assert len(syms) >= 35
    lib = ctypes.CDLL(LIB_PATH)
    missing = [s for s in sorted(syms) if not hasattr(lib, s)]
    assert not missing, missing
    # the Python binding declares exactly the header's entry points
    assert {n for n, _, _ in SIGNATURES} == syms


def test_abi_version_and_defaults():
    from paper_2110_08688_b200._lib import lib, mg_config
    assert lib().mg_abi_version() == 3
    assert ctypes.sizeof(mg_config) == 96  # mggcn.h layout (bias, dropout appended in ABI 3)
    c = mg_config()
    lib().mg_config_defaults(ctypes.byref(c))
    assert (c.lr, c.beta1, c.beta2, c.epsilon, c.epochs, c.seed) == (0.01, 0.9, 0.999, 1e-8, 100, 1)
    assert (c.bias, c.dropout) == (0, 0.0)


def test_config_validation_errors():
    with pytest.raises(R.ConfigError, match="at least one layer"):
        R.GcnConfig(layer_dims=[5]).validate()
    with pytest.raises(R.ConfigError, match="< 1"):
        R.GcnConfig(layer_dims=[5, 0, 3]).validate()
    with pytest.raises(R.ConfigError, match="negative epochs"):
        R.GcnConfig(layer_dims=[5, 3], epochs=-1).validate()
    with pytest.raises(R.ConfigError, match="unknown key 'bogus'"):
        R.parse_config({"hidden_dims": [8], "bogus": 1})
    cf = R.parse_config('{"hidden_dims": [256, 256], "lr": 0.05, "epochs": 3, "permute": true}')
    cfg = R.materialize_config(cf, 100, 47)
    assert cfg.layer_dims == [100, 256, 256, 47] and cfg.lr == 0.05 and cfg.permute and cfg.epochs == 3
    assert R.config_to_json(cfg)["layer_dims"] == [100, 256, 256, 47]


def test_synth_errors():
    with pytest.raises(R.ValueError, match="n >= 2"):
        R.synth_graph(1, 1.0, 0.7, 1)
    with pytest.raises(R.ValueError, match="infeasible"):
        R.synth_graph(10, 9.5, 0.7, 1)


def test_synth_bit_exact_vs_golden(golden):
    ds = R.synth_graph(300, 6.0, 0.7, 3, 12, 5)
    rp, ci, v = ds.graph
    assert np.array_equal(rp, golden["synth300_row_ptr"])
    assert np.array_equal(ci, golden["synth300_col_idx"])
    assert np.array_equal(v, golden["synth300_values"])
    assert np.array_equal(ds.features, golden["synth300_features"])
    assert np.array_equal(ds.labels, golden["synth300_labels"])
    c1 = R.synth_graph(2708, 3.9, 0.7, 1, 1433, 7)
    assert c1.nnz == 10566
    assert np.array_equal(c1.graph[0], golden["c1_row_ptr"]) and np.array_equal(c1.graph[1], golden["c1_col_idx"])
    import hashlib
    assert hashlib.sha256(c1.features.tobytes()).hexdigest() == golden["c1_features_sha256"].tobytes().decode()


def test_prepare_bit_exact_vs_golden(golden):
    ds = R.Dataset.from_arrays(golden["synth300_row_ptr"], golden["synth300_col_idx"], golden["synth300_values"],
                               golden["synth300_features"], golden["synth300_labels"])
    prep = R.prepare_data(ds, R.GcnConfig([12, 8, 5], seed=9, permute=True), 3)
    assert np.array_equal(prep.bounds, golden["prep300_bounds"])
    x, lab, m, pf = prep.rows_export(12)
    assert np.array_equal(pf, golden["prep300_perm"]) and np.array_equal(x, golden["prep300_features"])
    for d in (0, 1):
        for i in range(3):
            for j in range(3):
                rp, ci, v = prep.tile(d, i, j)
                assert np.array_equal(rp, golden[f"prep300_t{d}{i}{j}_rp"])
                assert np.array_equal(ci, golden[f"prep300_t{d}{i}{j}_ci"])
                assert np.array_equal(v, golden[f"prep300_t{d}{i}{j}_v"])


@pytest.mark.parametrize("P", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("permute", [False, True])
def test_prepare_matches_restatement(port32, P, permute):
    """Weighted, ragged graph (empty rows, empty parts for P > n/2) against the C restatement."""
    rng = np.random.default_rng(P * 10 + permute)
    n = 37
    dense = (rng.random((n, n)) < 0.15) * rng.uniform(0.1, 3.0, (n, n))
    dense[5, :] = 0  # an empty row
    dense[:, 7] = 0  # a zero-in-degree column (normalisation leaves it 0)
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum((dense != 0).sum(1))
    ci = np.nonzero(dense)[1].astype(np.int64)
    v = dense[dense != 0].astype(np.float32)
    x = rng.normal(size=(n, 3)).astype(np.float32)
    lab = rng.integers(0, 2, n).astype(np.int32)
    ds = R.Dataset.from_arrays(rp, ci, v, x, lab)
    prep = R.prepare_data(ds, R.GcnConfig([3, 2], seed=4, permute=permute), P)
    from oracle.pyoracle import Dataset as ODs
    pp = port32.prepare(ODs(n, rp, ci, v, x, lab), permute, 4, P)
    assert np.array_equal(prep.bounds, pp.bounds)
    for d in (0, 1):
        for i in range(P):
            for j in range(P):
                for a, b in zip(prep.tile(d, i, j), pp.tiles[d][i][j]):
                    assert np.array_equal(a, b), (d, i, j)


def test_prepare_only_rank_and_errors():
    ds = R.synth_graph(500, 8.0, 0.7, 5, 6, 3)
    cfg = R.GcnConfig([6, 4, 3], seed=2, permute=True)
    full = R.prepare_data(ds, cfg, 4)
    part = R.prepare_data(ds, cfg, 4, only_rank=2)
    for d in (0, 1):
        for j in range(4):
            for a, b in zip(full.tile(d, 2, j), part.tile(d, 2, j)):
                assert np.array_equal(a, b)
    with pytest.raises(R.ValueError, match="not built"):
        part.tile(0, 1, 0)
    with pytest.raises(R.ConfigError, match="layer_dims\\[0\\]=5"):
        R.prepare_data(ds, R.GcnConfig([5, 3]), 2)
    with pytest.raises(R.ValueError, match="P must be >= 1"):
        R.prepare_data(ds, cfg, 0)
    bad_mask = R.Dataset.from_arrays(*ds.graph, ds.features, ds.labels, train_mask=np.zeros(500, np.uint8))
    with pytest.raises(R.ValueError, match="training mask is empty"):
        R.prepare_data(bad_mask, cfg, 2)


def test_csr_validation():
    rp = np.array([0, 2, 3], np.int64)
    ci = np.array([1, 0, 0], np.int64)  # row 0 not increasing
    ds = R.Dataset.from_arrays(rp, ci, np.ones(3, np.float32), np.zeros((2, 1), np.float32), np.zeros(2, np.int32))
    with pytest.raises(R.ValueError, match="not strictly increasing"):
        ds.validate()


def test_aggregate_input_validation():
    from paper_2110_08688_b200._lib import lib, mg_config
    c = R.GcnConfig(layer_dims=[4, 8, 2])._c()
    assert c.aggregate_input == 1
    c.aggregate_input = 2
    assert lib().mg_config_validate(ctypes.byref(c)) == 6  # MG_CONFIG_ERROR
    d = mg_config()
    lib().mg_config_defaults(ctypes.byref(d))
    assert d.aggregate_input == 1 and d.spmm_mode == R.SPMM_FAST


def test_csr_validation_reports_the_first_violation():
    """CsrMatrix::validate (inc/sparse.hpp:37-54) scans rows in order: the first failing row wins, and an
    out-of-range column is named in the message — also when the parallel scan meets later rows first."""
    n = 200000
    rp = np.arange(n + 1, dtype=np.int64)
    ci = np.zeros(n, np.int64)
    ci[150000] = n + 5          # out of range late
    ci[3] = -1                  # out of range early: this one is reported
    ds = R.Dataset.from_arrays(rp, ci, np.ones(n, np.float32), np.zeros((n, 1), np.float32), np.zeros(n, np.int32))
    with pytest.raises(R.ValueError, match=r"^csr: col -1 out of range in row 3$"):
        ds.validate()
