"""Device partitioner (mg_prepare_device) against the host partitioner, which the CPU
suite pins bit-for-bit to the reference (tests/test_host.py): bounds, mask count, permuted rows and every
forward / backward tile (row pointers, local columns, normalised values) must be identical, for unit and
weighted graphs, permute on / off, P in {1, 2, 3, 8}, isolated vertices and P > n."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2110_08688_b200 import rowgcn as R  # noqa: E402


def weighted_graph(n, m, seed, isolated=0):
    rng = np.random.default_rng(seed)
    u = rng.integers(0, n - isolated, m)
    v = rng.integers(0, n - isolated, m)
    w = rng.uniform(0.1, 3.0, m).astype(np.float32)
    dense = {}
    for a, b, c in zip(u, v, w):
        dense[(int(a), int(b))] = dense.get((int(a), int(b)), np.float32(0)) + c
    keys = sorted(dense)
    rp = np.zeros(n + 1, np.int64)
    for a, _ in keys:
        rp[a + 1] += 1
    rp = np.cumsum(rp)
    ci = np.array([b for _, b in keys], np.int64)
    vals = np.array([dense[k] for k in keys], np.float32)
    x = rng.uniform(-1, 1, (n, 5)).astype(np.float32)
    lab = rng.integers(0, 3, n).astype(np.int32)
    mask = (rng.random(n) < 0.7).astype(np.uint8)
    mask[0] = 1
    return R.Dataset.from_arrays(rp, ci, vals, x, lab, mask)


def same_partition(ds, cfg, P):
    host = R.prepare_data(ds, cfg, P)
    dev = R.prepare_data(ds, cfg, P, device=0)
    assert list(host.bounds) == list(dev.bounds) and host.mask_count == dev.mask_count
    for a, b in zip(host.rows_export(cfg.layer_dims[0]), dev.rows_export(cfg.layer_dims[0])):
        assert np.array_equal(a, b)
    for d in range(2):
        for i in range(P):
            for j in range(P):
                for x, y in zip(host.tile(d, i, j), dev.tile(d, i, j)):
                    assert x.dtype == y.dtype and x.tobytes() == y.tobytes(), (d, i, j)


@pytest.mark.parametrize("P", [1, 2, 3, 8])
@pytest.mark.parametrize("permute", [False, True])
def test_device_partition_synth(P, permute):
    ds = R.synth_graph(5000, 12.0, 0.7, 3, 6, 4)
    same_partition(ds, R.GcnConfig([6, 8, 4], seed=11, permute=permute), P)


@pytest.mark.parametrize("P", [1, 3, 8])
def test_device_partition_weighted(P):
    ds = weighted_graph(700, 6000, 5, isolated=40)  # float weights: the column sums' order matters
    same_partition(ds, R.GcnConfig([5, 4, 3], seed=2, permute=True), P)


def test_device_partition_more_parts_than_rows():
    ds = weighted_graph(6, 20, 9)
    same_partition(ds, R.GcnConfig([5, 4, 3], seed=4, permute=True), 8)


def test_device_partition_trains_like_host():
    ds = R.synth_graph(20000, 20.0, 0.7, 1, 16, 5)
    cfg = R.GcnConfig([16, 32, 5], epochs=2, seed=1, permute=True)
    a = R.Group(cfg, R.prepare_data(ds, cfg, 1), 1, devices=[0])
    b = R.Group(cfg, R.prepare_data(ds, cfg, 1, device=0), 1, devices=[0])
    for g in (a, b):
        g.init_params()
    la = [a.train_step(t) for t in (1, 2)]
    lb = [b.train_step(t) for t in (1, 2)]
    assert la == lb
    a.close()
    b.close()
