"""Diagnostic: normwise deviations of W_G / W-after-Adam vs the C oracle for the production modes on a
hub-heavy graph (the smoke() configuration), with aggregate_input and hub segments toggled."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.pyoracle import Dataset as ODs, Port  # noqa: E402
from paper_2110_08688_b200 import rowgcn as R  # noqa: E402


def nw(a, b):
    return float(np.max(np.abs(a.astype(np.float64) - b)) / max(1e-30, np.max(np.abs(b))))


port = Port(np.float32)
n, dims = 4000, [40, 64, 32, 7]
ds = R.synth_graph(n, 40.0, 1.1, 5, dims[0], dims[-1])
rp, ci, v = ds.graph
ods = ODs(n, rp, ci, v, ds.features, ds.labels)
for agg in (True, False):
    for hr, seg in ((256, 64), (4096, 2048)):
        for gm in (R.GEMM_TF32X3, R.GEMM_EXACT):
            R.set_tuning("heavy_row", hr)
            R.set_tuning("fast_segment", seg)
            cfg = R.GcnConfig(dims, epochs=2, seed=4, permute=True, gemm_mode=gm, spmm_mode=R.SPMM_FAST,
                              aggregate_input=agg)
            prep = R.prepare_data(ds, cfg, 1)
            with R.Group(cfg, prep, 1, devices=[0]) as g:
                g.init_params()
                m = port.model(ods, dims, 1, seed=4, permute=True)
                lg = g.compute_gradients()
                rg = m.step(1, mode=1, dumps=True)
                wg = [nw(a, b) for a, b in zip(g.w_grads(), rg["w_grad"])]
            with R.Group(cfg, prep, 1, devices=[0]) as g:
                g.init_params()
                m = port.model(ods, dims, 1, seed=4, permute=True)
                ls = []
                for t in (1, 2):
                    ls.append((g.train_step(t), m.step(t, mode=0)["loss"]))
                w = [nw(a, b) for a, b in zip(g.params(), m.get_w())]
            print(f"agg={agg} heavy={hr} gemm={gm}: loss {lg:.7f}/{rg['loss']:.7f} WG {np.round(wg, 8)} "
                  f"losses {[(round(a, 7), round(b, 7)) for a, b in ls]} W {np.round(w, 8)}", flush=True)
R.set_tuning("heavy_row", 4096)
R.set_tuning("fast_segment", 2048)
