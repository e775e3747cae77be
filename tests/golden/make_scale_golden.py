"""Full-size parity fixtures from the UNMODIFIED reference (oracle/_ref, compiled by oracle/build_ref.sh).

Run in the build container (8+ cores, ~25 GB RAM for C4; /root/reference is not on the GPU box):

    python tests/golden/make_scale_golden.py [partition] [traj] [c4step] [c4s16step]

Writes, next to this script:
  scale_partition.json  sha256 of the reference's synth_graph output and of every prepare_data array
                        (permutation, permuted features / labels / mask, bounds, every forward and backward
                        tile) for the (config, P) pairs of tests/scale_common.PARTITION_CASES
                        (inc/dataset.hpp:287-334, inc/driver.hpp:87-117)
  scale_traj.npz        3-epoch train_run of C2 (full 169K-vertex arxiv shape) and of the products 1/16
                        sample: f64 and f32 losses, f32 and f64 final W, the sha256 of the f32 forward
                        activations and the f32 W_G / W after Adam of the teacher-forced step 1 (step_dump)
                        (inc/driver.hpp:140-206, inc/gcn.hpp:175-184)
  scale_c4step.npz      teacher-forced train_step(1) at full C4 (workers = 8): loss, W_G and W after Adam in
                        full; forward activations, loss gradient and H-grads on a row sample plus hub rows;
                        per-tensor max |x| and per-column sums (inc/gcn.hpp:175-184); the f64 build's W_G
  scale_c4s16step.npz   the same step on the products 1/16 sample from the f32 and the f64 reference
  scale_ranks.json      per-rank digests of prepare_data at papers shape, 1/64 scale, P = 8 (the rows and
                        tiles one rank of the job holds): pins the per-rank input path mg_synth_rank_*
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))
from oracle.pyoracle import Ref, make_cfg  # noqa: E402
from scale_common import (PARTITION_CASES, RANK_CASES, SCALE, c4_sample_rows, colsums, dataset_digest, sha,  # noqa: E402
                          tile_digest)

EPOCHS = 3


def log(*a):
    print(f"[{time.strftime('%H:%M:%S')}]", *a, flush=True)


def synth(ref, name, dtype=np.float32):
    c = SCALE[name]
    return ref.synth(c["n"], c["deg"], 0.7, 1, c["dims"][0], c["dims"][-1], dtype=dtype)


def partition(ref):
    out = {}
    by_cfg = {}
    for name, P in PARTITION_CASES:
        by_cfg.setdefault(name, []).append(P)
    for name, parts in by_cfg.items():
        ds = synth(ref, name)
        out[name] = {"dataset": dataset_digest(ds.row_ptr, ds.col_idx, ds.values, ds.features, ds.labels),
                     "n": ds.n, "nnz": ds.nnz, "parts": {}}
        log(name, "synth", ds.n, ds.nnz)
        for P in parts:
            cfg = make_cfg(SCALE[name]["dims"], seed=1, permute=True, overlap=P > 1)
            p = ref.prepare(ds, cfg, P)
            out[name]["parts"][str(P)] = {
                "bounds": [int(b) for b in p.bounds], "mask_count": int(p.mask_count),
                "perm_forward": sha(p.perm_forward), "features": sha(p.features), "labels": sha(p.labels),
                "mask": sha(p.mask),
                "tiles": {f"{d},{i},{j}": tile_digest(*p.tiles[d][i][j])
                          for d in (0, 1) for i in range(P) for j in range(P)},
                "nnz": {f"{d},{i},{j}": int(p.tiles[d][i][j][0][-1])
                        for d in (0, 1) for i in range(P) for j in range(P)}}
            log(name, "P", P, "done")
            del p
        del ds
    with open(os.path.join(HERE, "scale_partition.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


def traj(ref):
    g = {}
    for name in ("c2", "c4s16"):
        dims = SCALE[name]["dims"]
        cfg = make_cfg(dims, epochs=EPOCHS, seed=1, permute=True)
        d32 = synth(ref, name)
        r32 = ref.train_run(d32, cfg, 1)
        g[f"{name}_f32_loss"] = r32["loss"]
        g[f"{name}_f32_acc"] = r32["acc"]
        for l, w in enumerate(r32["final_w"]):
            g[f"{name}_f32_w{l}"] = w
        log(name, "f32", r32["loss"])
        dump = ref.step_dump(d32, make_cfg(dims, seed=1, permute=True), 1)
        for l, a in enumerate(dump["ahw_fwd"]):
            g[f"{name}_fwd_sha{l}"] = np.frombuffer(sha(np.asarray(a, np.float32)).encode(), np.uint8)
        for l in range(len(dims) - 1):  # teacher-forced step 1: W_G (well conditioned) and W after Adam
            g[f"{name}_f32_wgrad{l}"] = dump["w_grad"][l]
            g[f"{name}_f32_wafter{l}"] = dump["w_after"][l]
        del d32, dump
        d64 = synth(ref, name, np.float64)
        r64 = ref.train_run(d64, cfg, 1, np.float64)
        g[f"{name}_f64_loss"] = r64["loss"]
        for l, w in enumerate(r64["final_w"]):  # W after Adam is ill-conditioned: the reference's own f32
            g[f"{name}_f64_w{l}"] = w          # build is the yardstick (tests/test_gpu_scale.py)
        log(name, "f64", r64["loss"])
        del d64
    np.savez_compressed(os.path.join(HERE, "scale_traj.npz"), **g)


def step_stats(d, n, L, rows, prefix=""):
    """A teacher-forced step dump reduced to what is committed: loss, W_G, W after Adam in full; every
    row-indexed tensor on the sampled rows, with its max |x| and per-column sums / abs sums over all rows."""
    g = {f"{prefix}loss": np.array([d["loss"]])}
    for l in range(L):
        g[f"{prefix}wgrad{l}"] = d["w_grad"][l]
        g[f"{prefix}wafter{l}"] = d["w_after"][l]
    tensors = {f"fwd{l}": d["ahw_fwd"][l] for l in range(L)}
    tensors["loss_grad"] = d["loss_grad"]
    tensors.update({f"bwd{l}": d["ahw_bwd"][l] for l in range(L - 1)})  # H-grads (relu-masked)
    for k, a in tensors.items():
        a = np.asarray(a).reshape(n, -1)
        g[f"{prefix}{k}_rows"] = a[rows]
        g[f"{prefix}{k}_max"] = np.array([np.max(np.abs(a))], np.float64)
        s, sa = colsums(a)
        g[f"{prefix}{k}_colsum"] = s
        g[f"{prefix}{k}_colabs"] = sa
    return g


def sample_rows(ref, ds):
    fwd, _ = ref.random_permutation(ds.n, 1)
    deg_new = np.empty(ds.n, np.int64)
    deg_new[fwd] = np.diff(ds.row_ptr)
    return c4_sample_rows(ds.n, deg_new)


def c4step(ref):
    name = "c4"
    dims = SCALE[name]["dims"]
    L = len(dims) - 1
    ds = synth(ref, name)
    rows = sample_rows(ref, ds)
    log("c4 synth; sample rows", len(rows))
    cfg = make_cfg(dims, seed=1, permute=True, overlap=True)
    d = ref.step_dump(ds, cfg, 8)
    log("c4 step_dump loss", d["loss"])
    g = {"rows": rows, **step_stats(d, ds.n, L, rows)}
    del d, ds
    # the f64 build's W_G: the yardstick for how far the f32 reference itself is from exact (K = 306K
    # rows per canonical block)
    d64 = synth(ref, name, np.float64)
    r = ref.grad_run(d64, cfg, 8, np.float64)
    for l in range(L):
        g[f"f64_wgrad{l}"] = r["w_grad"][l]
    g["f64_loss"] = np.array([r["loss"]])
    log("c4 f64 grad_run loss", r["loss"])
    np.savez_compressed(os.path.join(HERE, "scale_c4step.npz"), **g)


def c4f64(ref):
    """Adds the f64 build's W_G and loss to an existing scale_c4step.npz (the f64 half of c4step)."""
    name = "c4"
    dims = SCALE[name]["dims"]
    path = os.path.join(HERE, "scale_c4step.npz")
    g = dict(np.load(path))
    cfg = make_cfg(dims, seed=1, permute=True, overlap=True)
    d64 = synth(ref, name, np.float64)
    r = ref.grad_run(d64, cfg, 8, np.float64)
    for l in range(len(dims) - 1):
        g[f"f64_wgrad{l}"] = r["w_grad"][l]
    g["f64_loss"] = np.array([r["loss"]])
    log("c4 f64 grad_run loss", r["loss"])
    np.savez_compressed(path, **g)


def c4s16step(ref):
    """The same teacher-forced step on the products 1/16 sample, dumped by the f32 AND the f64 reference:
    per-tensor distances of ours and of the f32 reference to the f64 one (tests/test_gpu_scale.py)."""
    name = "c4s16"
    dims = SCALE[name]["dims"]
    L = len(dims) - 1
    g = {}
    for dt, prefix in ((np.float32, ""), (np.float64, "f64_")):
        ds = synth(ref, name, dt)
        rows = sample_rows(ref, ds)
        d = ref.step_dump(ds, make_cfg(dims, seed=1, permute=True), 1, dt)
        g.update({"rows": rows, **step_stats(d, ds.n, L, rows, prefix)})
        log(name, dt.__name__, "step_dump loss", d["loss"])
    np.savez_compressed(os.path.join(HERE, "scale_c4s16step.npz"), **g)


def ranks(ref):
    """scale_ranks.json: for each (config, P) of RANK_CASES, the reference's whole-graph prepare_data cut
    into what one rank of a P-way job holds — per rank the bounds, its slices of the permuted features /
    labels / mask, and its forward and backward tile row (inc/driver.hpp:87-117) — plus the permutation."""
    out = {}
    for name, P in RANK_CASES:
        ds = synth(ref, name)
        log(name, "synth", ds.n, ds.nnz)
        d0 = SCALE[name]["dims"][0]
        cfg = make_cfg(SCALE[name]["dims"], seed=1, permute=True, overlap=True)
        p = ref.prepare(ds, cfg, P)
        feats = np.asarray(p.features, np.float32).reshape(ds.n, d0)
        e = {"n": ds.n, "nnz": ds.nnz, "P": P, "bounds": [int(b) for b in p.bounds],
             "mask_count": int(p.mask_count), "perm_forward": sha(p.perm_forward), "ranks": {}}
        for r in range(P):
            b0, b1 = int(p.bounds[r]), int(p.bounds[r + 1])
            e["ranks"][str(r)] = {
                "features": sha(feats[b0:b1]), "labels": sha(np.asarray(p.labels, np.int32)[b0:b1]),
                "mask": sha(np.asarray(p.mask, np.uint8)[b0:b1]),
                "tiles": {f"{d},{j}": tile_digest(*p.tiles[d][r][j]) for d in (0, 1) for j in range(P)},
                "nnz": {f"{d},{j}": int(p.tiles[d][r][j][0][-1]) for d in (0, 1) for j in range(P)}}
        out[f"{name}:{P}"] = e
        log(name, "P", P, "done")
        del p, ds, feats
    with open(os.path.join(HERE, "scale_ranks.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


def main():
    which = sys.argv[1:] or ["partition", "traj", "c4step", "c4s16step"]
    ref = Ref()
    ref.set_spmm_threads(max(1, (os.cpu_count() or 8)))
    for w in which:
        t = time.time()
        {"partition": partition, "traj": traj, "c4step": c4step, "c4f64": c4f64, "c4s16step": c4s16step,
         "ranks": ranks}[w](ref)
        log(w, f"{time.time() - t:.0f} s")


if __name__ == "__main__":
    main()
