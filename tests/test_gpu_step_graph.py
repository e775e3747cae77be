"""The training step replayed from a captured CUDA graph ("step_graph", one-worker groups) must be
bitwise the step launched kernel by kernel: same losses, accuracies, W hashes and Adam state, with the
per-step Adam constants patched into the graph, recaptures after a tuning change, and other group
calls (evaluation forward, gradient-only passes, writes) interleaved with replays."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
from paper_2110_08688_b200 import rowgcn as R  # noqa: E402

MODES = {
    "exact": dict(gemm_mode=R.GEMM_EXACT, spmm_mode=R.SPMM_EXACT),
    "production": dict(gemm_mode=R.GEMM_TF32X3, spmm_mode=R.SPMM_FAST, aggregate_input=True),
    "bias": dict(gemm_mode=R.GEMM_TF32X3, spmm_mode=R.SPMM_FAST, bias=True),
}


def cfg_layers(cfg):
    return len(cfg.layer_dims) - 1


def _set_graph(on):
    R.set_tuning("step_graph", 1 if on else 0)


def _run(ds, cfg, steps, on, between=None):
    _set_graph(on)
    try:
        prep = R.prepare_data(ds, cfg, 1)
        g = R.Group(cfg, prep, 1, devices=[0])
        g.init_params()
        out = []
        for t in range(1, steps + 1):
            loss = g.train_step(t)
            out.append((loss, g.last_accuracy, g.w_hash()))
            if between:
                between(g, t)
        state = [g.read(R.T_W, l) for l in range(cfg_layers(cfg))]
        state += [g.read(R.T_ADAM_M, l) for l in range(cfg_layers(cfg))]
        state += [g.read(R.T_ADAM_V, l) for l in range(cfg_layers(cfg))]
        replays, captures = g.graph_steps()
        g.close()
        return out, state, replays, captures
    finally:
        _set_graph(True)


@pytest.mark.parametrize("mode", sorted(MODES))
def test_graph_replay_bitwise(mode):
    ds = R.synth_graph(4000, 12.0, 0.7, 3, 24, 6)
    cfg = R.GcnConfig([24, 48, 32, 6], epochs=6, seed=5, permute=True, **MODES[mode])
    a, sa, ra, ca = _run(ds, cfg, 6, False)
    b, sb, rb, cb = _run(ds, cfg, 6, True)
    assert (ra, ca) == (0, 0)
    assert (rb, cb) == (6, 1)
    assert a == b
    for x, y in zip(sa, sb):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))


def test_graph_recapture_and_interleaved_calls():
    """A tuning change between steps recaptures; evaluation forwards and writes between replays are seen."""
    ds = R.synth_graph(3000, 10.0, 0.7, 4, 16, 5)
    cfg = R.GcnConfig([16, 40, 5], epochs=5, seed=2, permute=True, **MODES["production"])
    w_scale = np.float32(0.5)

    def between(g, t):
        if t == 2:
            R.set_tuning("heavy_row", 64)  # a different SpMM schedule from step 3 on (new capture)
        if t == 3:
            R.set_tuning("heavy_row", 4096)
        if t == 2:
            g.forward()  # evaluation pass on the same streams
        if t == 4:
            w0 = g.read(R.T_W, 0)
            g.write(R.T_W, 0, w0 * w_scale)

    try:
        a, sa, _, _ = _run(ds, cfg, 5, False, between)
        b, sb, rb, cb = _run(ds, cfg, 5, True, between)
    finally:
        R.set_tuning("heavy_row", 4096)
    assert rb == 5 and cb == 3  # captures at steps 1, 3 (heavy_row 64) and 4 (heavy_row back)
    assert a == b
    for x, y in zip(sa, sb):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))


def test_graph_not_used_with_profile_timeline_dropout():
    ds = R.synth_graph(1500, 8.0, 0.7, 1, 12, 4)
    cfg = R.GcnConfig([12, 16, 4], epochs=2, seed=1, permute=True, **MODES["production"])
    prep = R.prepare_data(ds, cfg, 1)
    g = R.Group(cfg, prep, 1, devices=[0])
    g.init_params()
    R.set_tuning("profile", 1)
    try:
        g.train_step(1)
    finally:
        R.set_tuning("profile", 0)
    assert g.graph_steps() == (0, 0)
    g.train_step(2)
    assert g.graph_steps() == (1, 1)
    k_graph = g.kernels_last_step()
    g.close()
    dcfg = R.GcnConfig([12, 16, 4], epochs=2, seed=1, permute=True, dropout=0.25, **MODES["production"])
    g = R.Group(dcfg, R.prepare_data(ds, dcfg, 1), 1, devices=[0])
    g.init_params()
    g.train_step(1)
    assert g.graph_steps() == (0, 0)
    g.close()
    assert k_graph > 0


def test_graph_async_steps_match_sync():
    """train_step_async replays back to back (no host wait between graphs) give the synchronous result."""
    ds = R.synth_graph(5000, 14.0, 0.7, 6, 32, 8)
    cfg = R.GcnConfig([32, 64, 8], epochs=8, seed=3, permute=True, **MODES["production"])
    prep = R.prepare_data(ds, cfg, 1)
    res = []
    for sync in (True, False):
        g = R.Group(cfg, prep, 1, devices=[0])
        g.init_params()
        for t in range(1, 9):
            if sync:
                g.train_step(t)
            else:
                g.train_step_async(t)
        g.sync()
        res.append((g.last_stats(), g.w_hash(), g.graph_steps()[0]))
        g.close()
    assert res[0] == res[1] and res[0][2] == 8
