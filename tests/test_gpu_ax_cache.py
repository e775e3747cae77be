"""Opt-in "ax_cache": under aggregate_input the layer-0 SpMM Â·X depends on the inputs only, so a group whose
ranks all live in this process computes it once and reuses it. The steps must be bitwise those of the
uncached step (stream path and graph replay, P = 1 and the in-process P = 2), a feature write must be seen
by the next step, and the cached step must launch fewer kernels."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
from paper_2110_08688_b200 import rowgcn as R  # noqa: E402

PROD = dict(gemm_mode=R.GEMM_TF32X3, spmm_mode=R.SPMM_FAST, aggregate_input=True)


def _run(ds, cfg, workers, steps, cache, graph, write_at=None):
    R.set_tuning("ax_cache", 1 if cache else 0)
    R.set_tuning("step_graph", 1 if graph else 0)
    try:
        prep = R.prepare_data(ds, cfg, workers)
        g = R.Group(cfg, prep, workers, devices=[0] * workers)
        g.init_params()
        out, kernels = [], []
        for t in range(1, steps + 1):
            loss = g.train_step(t)
            out.append((loss, g.last_accuracy, g.w_hash()))
            kernels.append(g.kernels_last_step())
            if write_at == t:  # new input features: the cached Â·X must be recomputed
                for r in range(workers):
                    x = g.read(R.T_X, 0, rank=r)
                    g.write(R.T_X, 0, x * np.float32(0.5), rank=r)
        w = [g.read(R.T_W, l) for l in range(len(cfg.layer_dims) - 1)]
        g.close()
        return out, w, kernels
    finally:
        R.set_tuning("ax_cache", 0)
        R.set_tuning("step_graph", 1)


@pytest.mark.parametrize("workers,graph", [(1, False), (1, True), (2, False)])
def test_ax_cache_bitwise(workers, graph):
    ds = R.synth_graph(4000, 12.0, 0.7, 3, 24, 6)
    cfg = R.GcnConfig([24, 48, 32, 6], epochs=6, seed=5, permute=True, **PROD)
    a, wa, ka = _run(ds, cfg, workers, 6, False, graph, write_at=3)
    b, wb, kb = _run(ds, cfg, workers, 6, True, graph, write_at=3)
    assert a == b
    for x, y in zip(wa, wb):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))
    # steps 1 and 4 compute Â·X (first step, after the write); the others reuse it
    for t in (2, 3, 5, 6):
        assert kb[t - 1] < ka[t - 1], (ka, kb)
    assert kb[0] == ka[0] and kb[3] == ka[3]


def test_ax_cache_needs_aggregate_input():
    ds = R.synth_graph(2000, 10.0, 0.7, 2, 16, 5)
    cfg = R.GcnConfig([16, 32, 5], epochs=3, seed=1, permute=True, gemm_mode=R.GEMM_TF32X3,
                      spmm_mode=R.SPMM_FAST, aggregate_input=False)
    a, _, ka = _run(ds, cfg, 1, 3, False, False)
    b, _, kb = _run(ds, cfg, 1, 3, True, False)
    assert a == b and ka == kb
