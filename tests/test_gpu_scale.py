"""Parity at the benchmarked sizes (the bench's reference-arm sample), against the
reference's own outputs pinned in tests/golden/scale_*.{json,npz} by tests/golden/make_scale_golden.py
(the compiled, unmodified reference; sha256 digests where arrays are too large to commit).

* partition: the synthetic graph, the permutation, permuted features / labels / mask, the bounds and every
  forward / backward tile of prepare_data are bit-identical for C2 (P = 1, 2), C3 (P = 1, 8) and C4
  (P = 1, 8) — host partitioner and device partitioner (inc/dataset.hpp:287-334, inc/driver.hpp:87-117);
* trajectories: 3 epochs of full C2 and of the products 1/16 sample in the production modes (TF32X3 GeMMs,
  FAST SpMM, aggregate_input) and in the EXACT modes, P = 1 and P = 2 (in-process transport): loss within
  1e-4 of the f64 reference, final W within 1e-4 (normwise) of the f32 reference; the EXACT forward is
  bitwise (sha256) equal to the reference's at C2;
* C4 teacher-forced step (production modes, real hub segments, 306K-row canonical W-grad blocks): forward
  activations, loss gradient and H-grads on sampled + hub rows and by per-column sums over all rows, W_G
  and W after Adam, all normwise <= 1e-4; loss rel <= 1e-4.
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from gpu_util import normwise  # noqa: E402
from scale_common import PARTITION_CASES, SCALE, colsums, dataset_digest, sha, tile_digest  # noqa: E402

from paper_2110_08688_b200 import rowgcn as R  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TOL = 1e-4


def golden_partition():
    with open(os.path.join(GOLD, "scale_partition.json")) as f:
        return json.load(f)


def synth(name):
    c = SCALE[name]
    return R.synth_graph(c["n"], c["deg"], 0.7, 1, c["dims"][0], c["dims"][-1])


def check_partition(prep, ds, gold, P):
    g = gold["parts"][str(P)]
    assert [int(b) for b in prep.bounds] == g["bounds"] and prep.mask_count == g["mask_count"]
    x, lab, m, pf = prep.rows_export(ds.d0)
    assert sha(pf) == g["perm_forward"] and sha(x) == g["features"]
    assert sha(lab) == g["labels"] and sha(m) == g["mask"]
    for d in (0, 1):
        for i in range(P):
            for j in range(P):
                assert tile_digest(*prep.tile(d, i, j)) == g["tiles"][f"{d},{i},{j}"], (d, i, j)


@pytest.mark.parametrize("name,P", PARTITION_CASES)
def test_partition_bit_identical(name, P):
    gold = golden_partition()[name]
    ds = synth(name)
    rp, ci, v = ds.graph
    assert dataset_digest(rp, ci, v, ds.features, ds.labels) == gold["dataset"]
    cfg = R.GcnConfig(SCALE[name]["dims"], seed=1, permute=True, overlap=P > 1)
    check_partition(R.prepare_data(ds, cfg, P), ds, gold, P)  # host partitioner
    check_partition(R.prepare_data(ds, cfg, P, device=0), ds, gold, P)  # device partitioner


MODES = {"production": dict(gemm_mode=R.GEMM_TF32X3, spmm_mode=R.SPMM_FAST, aggregate_input=True),
         "exact": dict(gemm_mode=R.GEMM_EXACT, spmm_mode=R.SPMM_EXACT)}


@pytest.fixture(scope="module")
def traj():
    return np.load(os.path.join(GOLD, "scale_traj.npz"))


@pytest.mark.parametrize("name", ["c2", "c4s16"])
@pytest.mark.parametrize("mode", ["production", "exact"])
@pytest.mark.parametrize("P", [1, 2])
def test_trajectory(traj, name, mode, P):
    dims = SCALE[name]["dims"]
    ds = synth(name)
    cfg = R.GcnConfig(dims, epochs=3, seed=1, permute=True, overlap=P > 1, **MODES[mode])
    art = R.train_run(ds, cfg, R.TrainOptions(workers=P, devices=[0] * P,
                                              transport=R.TRANSPORT_NCCL if P == 1 else R.TRANSPORT_LOCAL))
    r64 = traj[f"{name}_f64_loss"]
    rel = [abs(a - b) / abs(b) for a, b in zip(art.epoch_loss, r64)]
    assert max(rel) <= TOL, rel
    dev = [normwise(art.final_w[l], traj[f"{name}_f32_w{l}"]) for l in range(len(dims) - 1)]
    assert max(dev) <= TOL, dev


@pytest.mark.parametrize("P", [1, 2])
def test_c2_exact_forward_bitwise(traj, P):
    dims = SCALE["c2"]["dims"]
    ds = synth("c2")
    cfg = R.GcnConfig(dims, seed=1, permute=True, overlap=P > 1, **MODES["exact"])
    prep = R.prepare_data(ds, cfg, P)
    with R.Group(cfg, prep, P, devices=[0] * P, transport=R.TRANSPORT_NCCL if P == 1 else R.TRANSPORT_LOCAL) as g:
        g.init_params()
        g.forward()
        for l in range(len(dims) - 1):
            a = np.concatenate([g.read(R.T_AHW, l, r) for r in range(P)], axis=0)
            assert sha(a) == bytes(traj[f"c2_fwd_sha{l}"]).decode(), f"layer {l}"


@pytest.fixture(scope="module")
def c4():
    return np.load(os.path.join(GOLD, "scale_c4step.npz"))


def check_rows(a, c4, key):
    """Sampled rows normwise against the full tensor's max |x|, plus per-column sums over every row."""
    rows = c4["rows"]
    d_rows = float(np.max(np.abs(a[rows].astype(np.float64) - c4[f"{key}_rows"])) / c4[f"{key}_max"][0])
    s, _ = colsums(a)
    d_cols = float(np.max(np.abs(s - c4[f"{key}_colsum"]) / np.maximum(c4[f"{key}_colabs"], 1e-30)))
    return d_rows, d_cols


def test_c4_teacher_forced_step(c4):
    dims = SCALE["c4"]["dims"]
    L = len(dims) - 1
    ds = synth("c4")
    cfg = R.GcnConfig(dims, seed=1, permute=True, **MODES["production"])
    prep = R.prepare_data(ds, cfg, 1, device=0)
    report = {}
    with R.Group(cfg, prep, 1, devices=[0]) as g:
        g.init_params()
        g.forward()
        for l in range(L):
            report[f"fwd{l}"] = check_rows(g.read(R.T_AHW, l), c4, f"fwd{l}")
    with R.Group(cfg, prep, 1, devices=[0]) as g:
        g.init_params()
        loss = g.compute_gradients()
        report["loss"] = abs(loss - c4["loss"][0]) / abs(c4["loss"][0])
        for l in range(L):
            report[f"wgrad{l}"] = normwise(g.read(R.T_WGRAD, l), c4[f"wgrad{l}"])
        report["loss_grad"] = check_rows(g.read(R.T_AHW, L - 1), c4, "loss_grad")
        for l in range(L - 1):
            report[f"bwd{l}"] = check_rows(g.read(R.T_AHW, l), c4, f"bwd{l}")
    with R.Group(cfg, prep, 1, devices=[0]) as g:
        g.init_params()
        g.train_step(1)
        for l in range(L):
            report[f"wafter{l}"] = normwise(g.read(R.T_W, l), c4[f"wafter{l}"])
    print(json.dumps(report))
    worst = max(max(v) if isinstance(v, tuple) else v for v in report.values())
    assert worst <= TOL, report
