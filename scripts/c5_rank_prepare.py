"""Full papers-shaped C5 (111,059,956 vertices, avg degree 28.8, [128,128,128,172]) at P = 8: ONE rank's
partition through the per-rank input path (mg_synth_rank_*), as one process of an 8-GPU job would build
it — timed per phase, with the process's peak host RSS. A lone process derives every vertex's degree by
P block passes (under torchrun the ranks all-gather them instead: bench.py / paper_2110_08688_b200.torchdist).

    python scripts/c5_rank_prepare.py [rank] [P] [--scale K]   (K: 1/K of the vertices)
"""
import json
import os
import resource
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_08688_b200 import rowgcn as R  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
rank = int(args[0]) if args else 0
P = int(args[1]) if len(args) > 1 else 8
scale = int(sys.argv[sys.argv.index("--scale") + 1]) if "--scale" in sys.argv else 1
n = 111059956 // scale
dims = [128, 128, 128, 172]
cfg = R.GcnConfig(dims, seed=1, permute=True, overlap=True)


def rss_gb():
    return resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6


t0 = time.time()
h = R.SynthRank(n, 28.8, 0.7, 1, dims[0], dims[-1], cfg, P, rank)
t1 = time.time()
deg = np.empty(n, np.int32)
for b in range(P):
    deg[b * n // P:(b + 1) * n // P] = h.block_degrees(b)
t2 = time.time()
prep = h.finish(deg)
t3 = time.time()
del h
nnz = [prep.tile(0, rank, j)[0][-1] for j in range(P)]
out = {"n": n, "P": P, "rank": rank, "stubs_and_rows_s": round(t1 - t0, 1), "degree_passes_s": round(t2 - t1, 1),
       "tiles_s": round(t3 - t2, 1), "total_s": round(t3 - t0, 1), "rank_nnz": int(sum(nnz)),
       "rank_rows": int(prep.bounds[rank + 1] - prep.bounds[rank]), "stage_nnz": [int(z) for z in nnz],
       "max_degree": int(deg.max()), "edges": int(deg.astype(np.int64).sum()), "peak_rss_gb": round(rss_gb(), 2),
       "host_threads": os.cpu_count()}
print(json.dumps(out))
