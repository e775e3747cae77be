"""The C++ drop-in (include/mggcn/rowgcn.hpp) driving the device path end to end on the GPU, and the
reference-style driver behaviours (on_epoch, checkpoints, collect_logits equivariance)."""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

from paper_2110_08688_b200 import rowgcn as R  # noqa: E402


def test_cpp_dropin_trains(tmp_path):
    exe = tmp_path / "train_products"
    lib = os.path.join(ROOT, "paper_2110_08688_b200")
    r = subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "examples", "train_products.cpp"), "-L", lib, "-lmggcn",
                        f"-Wl,-rpath,{lib}", "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    run = subprocess.run([str(exe), "20000", "3", "1"], capture_output=True, text=True, timeout=300)
    assert run.returncode == 0, run.stderr
    lines = [ln for ln in run.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 3
    import json
    losses = [json.loads(ln)["loss"] for ln in lines]
    # same run through the Python mirror (same library, same defaults) gives the same trajectory
    ds = R.synth_graph(20000, 50.6, 0.7, 1, 100, 47)
    art = R.train_run(ds, R.GcnConfig([100, 256, 256, 47], epochs=3, permute=True), R.TrainOptions(devices=[0]))
    np.testing.assert_allclose(losses, art.epoch_loss, rtol=1e-6)
    n_events = int(next(ln for ln in run.stdout.splitlines() if ln.startswith("timeline:")).split()[1])
    assert n_events == len(art.timeline) > 0


def test_on_epoch_and_logit_equivariance():
    """tests/test_gcn.cpp:370-393: permutation changes the layout, not the problem."""
    ds = R.synth_graph(700, 8.0, 0.6, 17, 4, 2)
    cfg = R.GcnConfig([4, 6, 2], epochs=4, seed=5, gemm_mode=R.GEMM_EXACT, spmm_mode=R.SPMM_EXACT)
    seen = []
    plain = R.train_run(ds, cfg, R.TrainOptions(workers=2, devices=[0, 0], collect_logits=True,
                                                on_epoch=lambda *a: seen.append(a),
                                                transport=R.TRANSPORT_LOCAL))
    assert [s[0] for s in seen] == [1, 2, 3, 4]
    cfg.permute = True
    perm = R.train_run(ds, cfg, R.TrainOptions(workers=2, devices=[0, 0], collect_logits=True,
                                               transport=R.TRANSPORT_LOCAL))
    np.testing.assert_allclose(plain.epoch_loss, perm.epoch_loss, rtol=1e-5)
    pf = R.prepare_data(ds, cfg, 2).rows_export(4)[3]
    np.testing.assert_allclose(plain.logits, perm.logits[pf], rtol=1e-4, atol=1e-5)
