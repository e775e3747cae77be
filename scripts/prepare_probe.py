"""Host vs device partitioner time (and bit-equality of a sample of tiles) at C4 and scaled-C5 shapes."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402,F401  (before libmggcn)
from paper_2110_08688_b200 import rowgcn as R  # noqa: E402

for name, n, deg, dims in [("c4", 2449029, 50.6, [100, 256, 256, 47]),
                           ("c5/8", 111059956 // 8, 28.8, [128, 128, 128, 172]),
                           ("c5/4", 111059956 // 4, 28.8, [128, 128, 128, 172])]:
    t0 = time.time()
    ds = R.synth_graph(n, deg, 0.7, 1, dims[0], dims[-1])
    t1 = time.time()
    cfg = R.GcnConfig(dims, epochs=1, seed=1, permute=True)
    for P in (1, 8):
        a = time.time()
        dev = R.prepare_data(ds, cfg, P, device=0)
        b = time.time()
        host = R.prepare_data(ds, cfg, P) if name != "c5/4" else None
        c = time.time()
        same = "n/a"
        if host is not None:
            same = all(x.tobytes() == y.tobytes() for d in range(2) for (i, j) in ((0, 0), (P - 1, P - 1), (0, P - 1))
                       for x, y in zip(host.tile(d, i, j), dev.tile(d, i, j)))
        print(f"{name} n={n} nnz={ds.nnz} P={P}: synth {t1 - t0:.1f} s, device prepare {b - a:.2f} s, "
              f"host prepare {c - b:.2f} s, sampled tiles identical: {same}", flush=True)
        del dev, host
    del ds
