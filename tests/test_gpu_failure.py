"""Failure semantics of the device group, after the reference's DeviceGroup (proj/src/collectives.cpp:33-52,
tests/test_collectives.cpp:136-151): abort() from another thread and a watchdog on every host wait wake the
waiter with ShutdownError; the aborted group refuses further work and can still be destroyed. A peer that
never joins the NCCL communicator is the test_collectives "worker that never arrives" case. The stall is
injected with the "debug_stall_us" test hook (a spin kernel at step start) on the in-process transport."""
import threading
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2110_08688_b200 import rowgcn as R  # noqa: E402


@pytest.fixture
def tuning():
    yield R.set_tuning
    for k in ("debug_stall_us", "watchdog_ms", "nccl_single"):
        R.set_tuning(k, 0)


def local_group(P=2):
    ds = R.synth_graph(500, 6.0, 0.6, 3, 8, 4)
    cfg = R.GcnConfig([8, 8, 4], seed=2, permute=True, overlap=True)
    prep = R.prepare_data(ds, cfg, P)
    g = R.Group(cfg, prep, P, devices=[0] * P, transport=R.TRANSPORT_LOCAL)
    g.init_params()
    return g


def test_watchdog_aborts_a_stalled_step(tuning):
    g = local_group()
    g.train_step(1)  # healthy
    tuning("debug_stall_us", 3_000_000)
    tuning("watchdog_ms", 300)
    t0 = time.time()
    with pytest.raises(R.ShutdownError, match="watchdog_ms=300"):
        g.train_step(2)
    assert time.time() - t0 < 2.5  # woken by the watchdog, not by the stall ending
    tuning("debug_stall_us", 0)
    with pytest.raises(R.ShutdownError, match="device group aborted"):
        g.train_step(3)
    with pytest.raises(R.ShutdownError):
        g.read(R.T_W, 0)
    g.close()  # destroy still releases everything (after the stall kernel drains)


def test_abort_from_another_thread(tuning):
    g = local_group()
    tuning("debug_stall_us", 2_000_000)
    th = threading.Timer(0.1, g.abort)
    th.start()
    t0 = time.time()
    with pytest.raises(R.ShutdownError, match="abort requested"):
        g.train_step(1)
    th.join()
    assert time.time() - t0 < 1.5
    g.close()


def test_nccl_peer_that_never_arrives(tuning):
    """world = 2 with only rank 0 present: communicator creation would wait forever; the watchdog aborts it."""
    tuning("watchdog_ms", 1500)
    ds = R.synth_graph(300, 5.0, 0.6, 3, 4, 2)
    cfg = R.GcnConfig([4, 4, 2], seed=1)
    prep = R.prepare_data(ds, cfg, 2, only_rank=0)
    t0 = time.time()
    with pytest.raises(R.ShutdownError, match="did not complete"):
        R.Group(cfg, prep, 2, local_ranks=[0], devices=[0], nccl_id=R.nccl_unique_id())
    assert time.time() - t0 < 30


@pytest.mark.parametrize("mode", ["exact", "production"])
def test_nccl_collectives_single_rank(tuning, mode):
    """The non-blocking NCCL enqueue + settle path executed for real on one device (a one-rank communicator:
    in-place broadcast, one-rank all-reduce): the trajectory is bitwise the communicator-free one."""
    kw = (dict(gemm_mode=R.GEMM_EXACT, spmm_mode=R.SPMM_EXACT) if mode == "exact" else {})
    ds = R.synth_graph(3000, 8.0, 0.7, 11, 20, 5)
    cfg = R.GcnConfig([20, 24, 5], epochs=3, seed=2, permute=True, **kw)
    base = R.train_run(ds, cfg, R.TrainOptions(devices=[0]))
    tuning("nccl_single", 1)
    tuning("watchdog_ms", 60_000)
    nccl = R.train_run(ds, cfg, R.TrainOptions(devices=[0], transport=R.TRANSPORT_NCCL))
    assert nccl.epoch_loss == base.epoch_loss and nccl.w_hashes == base.w_hashes
    assert all(np.array_equal(a, b) for a, b in zip(nccl.final_w, base.final_w))
