"""Timeline from CUDA events and bench-spmm (row 4): the device trainer records one
TimelineEvent per task the reference submits (inc/collectives.hpp:24-34), exported in the reference
schema; the exported files pass the reference's OWN load_timeline / audit_timeline / audit_staged_run
(oracle/_ref) and its runtime_breakdown agrees with ours; the task structure matches the reference
trainer's own timeline except the fused ReLU / relu_backward tasks."""
import collections
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
from gpu_util import bits_equal  # noqa: E402

from paper_2110_08688_b200 import rowgcn as R  # noqa: E402

FUSED = {"relu", "relu_bwd"}  # fused into the SpMM / hgrad epilogues: no task of their own here


def structure(events):
    return collections.Counter((e.worker, e.lane, e.stage, e.kind, e.op) for e in events if e.op not in FUSED)


@pytest.mark.parametrize("P,overlap", [(1, False), (2, True), (2, False), (4, True)])
def test_train_timeline_passes_reference_audits(ref, tmp_path, P, overlap):
    from oracle.pyoracle import make_cfg
    ds = R.synth_graph(3000, 8.0, 0.7, 3, 12, 5)
    dims = [12, 16, 5]
    cfg = R.GcnConfig(dims, epochs=2, seed=2, permute=True, overlap=overlap, gemm_mode=R.GEMM_EXACT,
                      spmm_mode=R.SPMM_EXACT)
    art = R.train_run(ds, cfg, R.TrainOptions(workers=P, devices=[0] * P,
                                              transport=R.TRANSPORT_NCCL if P == 1 else R.TRANSPORT_LOCAL))
    ev = art.timeline
    assert ev and all(e.t_end_us >= e.t_start_us for e in ev)
    R.audit_timeline(ev)
    path = tmp_path / "tl.json"
    R.export_timeline(path, ev)
    assert R.load_timeline(path) == ev
    count, theirs = ref.timeline_check(path)  # the reference's own parser + audit
    assert count == len(ev)
    ours = R.runtime_breakdown(ev).to_json()["totals_us"]
    for k in theirs:
        assert ours[k] == pytest.approx(theirs[k], rel=1e-12, abs=1e-9)
    assert ours["spmm"] > 0 and ours["gemm"] > 0 and ours["loss"] > 0 and ours["adam"] > 0
    # task structure: the reference trainer's own timeline on the same data and config
    rds = ref.synth(3000, 8.0, 0.7, 3, 12, 5)
    ref.train_timeline(rds, make_cfg(dims, epochs=2, seed=2, permute=True, overlap=overlap), P, tmp_path / "ref.json")
    assert structure(R.load_timeline(tmp_path / "ref.json")) == structure(ev)


def test_audit_rejects_what_the_reference_rejects(ref, tmp_path):
    ds = R.synth_graph(2000, 6.0, 0.7, 1, 8, 3)
    art = R.train_run(ds, R.GcnConfig([8, 8, 3], epochs=1, seed=1, permute=True, overlap=True),
                      R.TrainOptions(workers=2, devices=[0, 0], transport=R.TRANSPORT_LOCAL))
    ev = art.timeline
    spmm = next(e for e in ev if e.kind == "spmm" and e.deps)
    dep = next(e for e in ev if e.task == spmm.deps[0])
    bad = [R.TimelineEvent(**{**e.__dict__}) for e in ev]
    victim = next(e for e in bad if e.task == spmm.task)
    victim.t_start_us = dep.t_end_us - 1.0  # starts before its broadcast finished
    victim.t_end_us = max(victim.t_end_us, victim.t_start_us)
    path = tmp_path / "bad.json"
    R.export_timeline(path, bad)
    with pytest.raises(R.ValueError):
        R.audit_timeline(bad)
    from oracle.pyoracle import OracleError
    with pytest.raises(OracleError):
        ref.timeline_check(path)


@pytest.mark.parametrize("P,overlap", [(1, False), (2, True), (3, False), (4, True), (4, False)])
def test_bench_spmm_staged_rules_and_result(ref, port32, tmp_path, P, overlap):
    """bench-spmm (proj/tools/main.cpp:120-178): one staged SpMM; the staged-run audit of the reference
    holds, the stage CSV has one line per (stage, worker), and in exact mode the result is bitwise the
    reference's monolithic spmm of the permuted, normalised, transposed graph."""
    from oracle.pyoracle import make_cfg
    ds = R.synth_graph(2500, 10.0, 0.7, 7, 40, 2)
    tl, csv = tmp_path / "spmm.json", tmp_path / "stages.csv"
    res = R.bench_spmm(ds, workers=P, overlap=overlap, timeline_path=str(tl), stage_csv=str(csv),
                       devices=[0] * P, transport=R.TRANSPORT_NCCL if P == 1 else R.TRANSPORT_LOCAL,
                       spmm_mode=R.SPMM_EXACT)
    ref.timeline_check(tl, world=P, overlapped=overlap and P > 1)
    lines = open(csv).read().splitlines()
    assert lines[0] == "stage,worker,comm_us,comp_us" and len(lines) == 1 + P * P
    assert res["width"] == 40 and res["workers"] == P and res["nnz"] == ds.nnz
    assert res["bytes_broadcast"] == (2500 * 40 * 4 if P > 1 else 0)
    # monolithic reference: fwd tiles of the reference's own prepare_data, reassembled per row block
    rprep = ref.prepare(ref.synth(2500, 10.0, 0.7, 7, 40, 2), make_cfg([40, 40], seed=1, permute=True), P)
    x = rprep.features
    outs = []
    for i in range(P):
        rows = rprep.bounds[i + 1] - rprep.bounds[i]
        rp = np.zeros(rows + 1, np.int64)
        ci, v = [], []
        for r in range(rows):
            for j in range(P):
                trp, tci, tv = rprep.tiles[0][i][j]
                ci.extend((tci[trp[r]:trp[r + 1]] + rprep.bounds[j]).tolist())
                v.extend(tv[trp[r]:trp[r + 1]].tolist())
            rp[r + 1] = len(ci)
        outs.append(port32.spmm(rows, 2500, rp, np.array(ci, np.int64), np.array(v, np.float32), x))
    assert bits_equal(res["out"], np.concatenate(outs, axis=0))


def test_bench_spmm_fast_close_to_exact():
    ds = R.synth_graph(4000, 20.0, 0.7, 9, 256, 2)
    a = R.bench_spmm(ds, workers=2, devices=[0, 0], transport=R.TRANSPORT_LOCAL, spmm_mode=R.SPMM_EXACT)
    b = R.bench_spmm(ds, workers=2, devices=[0, 0], transport=R.TRANSPORT_LOCAL, spmm_mode=R.SPMM_FAST)
    assert np.max(np.abs(a["out"] - b["out"])) <= 1e-5 * np.max(np.abs(a["out"]))
    assert b["device_us"] > 0 and b["wall_us"] > 0
