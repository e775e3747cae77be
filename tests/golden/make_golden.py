"""Generates tests/golden/*.npz from the UNMODIFIED reference compiled by oracle/build_ref.sh.

Run in the build container (needs oracle/_ref/librowgcn_ref.so):  python tests/golden/make_golden.py
Every array here is the reference's own output on seeded inputs; tests/test_oracle.py pins the C
restatement (oracle/oracle.c) against these fixtures and the device tests reuse them.
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.pyoracle import Ref, make_cfg  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def random_csr(rng, n, density, lo=-1.0, hi=1.0):
    m = rng.random((n, n)) < density
    vals = rng.uniform(lo, hi, size=(n, n))
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum(m.sum(1))
    ci = np.nonzero(m)[1].astype(np.int64)
    v = vals[m]
    return rp, ci, v


def main():
    ref = Ref()
    g = {}
    # ---- KATs (inc/rng.hpp, inc/partition.hpp; tests/test_partition.cpp:50-95)
    g["perm_8_7_inverse"] = ref.random_permutation(8, 7)[1]
    g["perm_2708_1_forward"] = ref.random_permutation(2708, 1)[0]
    for n, p in [(10, 4), (8, 8), (5, 8), (2449029, 8), (169343, 2), (232965, 4)]:
        g[f"partition_{n}_{p}"] = ref.uniform_partition(n, p)
    # ---- synth graphs: a small one in full, the C1 (Cora-shaped) one by hash
    small = ref.synth(300, 6.0, 0.7, 3, 12, 5)
    for k in ("row_ptr", "col_idx", "values", "features", "labels"):
        g[f"synth300_{k}"] = getattr(small, k)
    c1 = ref.synth(2708, 3.9, 0.7, 1, 1433, 7)
    g["c1_row_ptr"] = c1.row_ptr
    g["c1_col_idx"] = c1.col_idx
    g["c1_labels"] = c1.labels
    g["c1_features_sha256"] = np.frombuffer(sha(c1.features).encode(), np.uint8)
    # ---- prepared tiles (small graph, P=3, permuted)
    prep = ref.prepare(small, make_cfg([12, 8, 5], seed=9, permute=True), 3)
    g["prep300_bounds"] = prep.bounds
    g["prep300_perm"] = prep.perm_forward
    g["prep300_features"] = prep.features
    for d in (0, 1):
        for i in range(3):
            for j in range(3):
                rp, ci, v = prep.tiles[d][i][j]
                g[f"prep300_t{d}{i}{j}_rp"] = rp
                g[f"prep300_t{d}{i}{j}_ci"] = ci
                g[f"prep300_t{d}{i}{j}_v"] = v
    # ---- kernels on random inputs (f32 and f64)
    rng = np.random.default_rng(2024)
    for k in range(4):
        n = int(rng.integers(20, 120))
        w = int(rng.integers(1, 40))
        rp, ci, v = random_csr(rng, n, float(rng.uniform(0.02, 0.4)))
        for dt, s in ((np.float32, "f32"), (np.float64, "f64")):
            h = rng.uniform(-1, 1, (n, w)).astype(dt)
            o0 = rng.uniform(-1, 1, (n, w)).astype(dt)
            g[f"spmm{k}_{s}_rp"], g[f"spmm{k}_{s}_ci"], g[f"spmm{k}_{s}_v"] = rp, ci, v.astype(dt)
            g[f"spmm{k}_{s}_h"], g[f"spmm{k}_{s}_o0"] = h, o0
            g[f"spmm{k}_{s}_out"] = ref.spmm(n, n, rp, ci, v.astype(dt), h)
            g[f"spmm{k}_{s}_acc"] = ref.spmm(n, n, rp, ci, v.astype(dt), h, accumulate=True, out=o0)
    for k, (ta, tb) in enumerate([(False, False), (True, False), (False, True), (True, True)]):
        m_, k_, n_ = (int(x) for x in rng.integers(1, 40, 3))
        for dt, s in ((np.float32, "f32"), (np.float64, "f64")):
            a = rng.uniform(-1, 1, (k_, m_) if ta else (m_, k_)).astype(dt)
            a[rng.random(a.shape) < 0.2] = 0  # exercise the zero-skip (inc/dense.hpp:165, :177)
            b = rng.uniform(-1, 1, (n_, k_) if tb else (k_, n_)).astype(dt)
            g[f"gemm{k}_{s}_a"], g[f"gemm{k}_{s}_b"] = a, b
            g[f"gemm{k}_{s}_out"] = ref.gemm(a, b, ta, tb)
    for dt, s in ((np.float32, "f32"), (np.float64, "f64")):
        logits = rng.normal(0, 3, (64, 7)).astype(dt)
        labels = rng.integers(0, 7, 64).astype(np.int32)
        mask = (rng.random(64) < 0.7).astype(np.uint8)
        ls, grad = ref.softmax_xent_sum(logits, labels, mask, int(mask.sum()) + 3)
        g[f"xent_{s}_logits"], g[f"xent_{s}_labels"], g[f"xent_{s}_mask"] = logits, labels, mask
        g[f"xent_{s}_loss"], g[f"xent_{s}_grad"] = np.array([ls]), grad
        w, gr, m, vv = (rng.normal(0, 1, 50).astype(dt) for _ in range(4))
        vv = np.abs(vv)
        outs = ref.adam(w, gr, m, vv, 3, lr=0.05)
        for nm, arr in zip("wgmv", (w, gr, m, vv)):
            g[f"adam_{s}_{nm}_in"] = arr
        for nm, arr in zip("wgmv", outs):
            g[f"adam_{s}_{nm}_out"] = arr
    # ---- model trajectories: C1 (Cora-shaped) [1433,16,7], 5 epochs, both dtypes, permute on/off
    c1_64 = ref.synth(2708, 3.9, 0.7, 1, 1433, 7, dtype=np.float64)
    for perm in (False, True):
        cfg = make_cfg([1433, 16, 7], epochs=5, seed=1, permute=perm)
        r = ref.train_run(c1, cfg, 1)
        g[f"c1_f32_perm{int(perm)}_loss"] = r["loss"]
        g[f"c1_f32_perm{int(perm)}_acc"] = r["acc"]
        g[f"c1_f32_perm{int(perm)}_hash"] = r["w_hashes"][:, 0]
        r = ref.train_run(c1_64, cfg, 1, dtype=np.float64)
        g[f"c1_f64_perm{int(perm)}_loss"] = r["loss"]
    # P-invariance of the W trajectory (tests/test_gcn.cpp:323-348)
    for P in (2, 4, 8):
        r = ref.train_run(c1, make_cfg([1433, 16, 7], epochs=5, seed=1, permute=True, overlap=True), P)
        g[f"c1_f32_perm1_P{P}_hash"] = r["w_hashes"][:, 0]
        g[f"c1_f32_perm1_P{P}_loss"] = r["loss"]
    # ---- teacher-forced step dump on the small graph, 3 layers, P=2 (all intermediates)
    cfg = make_cfg([12, 8, 6, 5], epochs=1, seed=5, permute=True, overlap=True)
    d = ref.step_dump(small, cfg, 2)
    g["dump300_loss"] = np.array([d["loss"]])
    for l in range(3):
        g[f"dump300_ahw_fwd{l}"] = d["ahw_fwd"][l]
        g[f"dump300_ahw_bwd{l}"] = d["ahw_bwd"][l]
        g[f"dump300_wgrad{l}"] = d["w_grad"][l]
        g[f"dump300_wafter{l}"] = d["w_after"][l]
    g["dump300_loss_grad"] = d["loss_grad"]
    np.savez_compressed(os.path.join(OUT, "reference_golden.npz"), **g)
    print("wrote", os.path.join(OUT, "reference_golden.npz"), len(g), "arrays")


if __name__ == "__main__":
    main()
