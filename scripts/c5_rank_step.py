"""One rank of the papers-shaped C5 job at P = 8 (111 M vertices, 3.2 B edges, [128, 128, 128, 172]) on ONE
B200: rank `r`'s real partition (mg_synth_rank_*, bit-identical to that row block of the reference's
prepare_data) in a group created with the measurement-only solo transport (mggcn.h MG_TRANSPORT_SOLO: the
broadcasts / all-reduces are skipped, the receive buffers keep what they hold). Times the rank's device
work per training step (CUDA events, after warm-up) with the per-kind breakdown, for stage folding off and
in groups of 2 and 4 — the compute side of the 8-GPU epoch; the exchange adds n_p-row blocks over NVLink.

    python scripts/c5_rank_step.py [rank] [--scale K] [--steps S]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import numpy as np  # noqa: E402
from paper_2110_08688_b200 import rowgcn as R  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
rank = int(args[0]) if args else 0
scale = int(sys.argv[sys.argv.index("--scale") + 1]) if "--scale" in sys.argv else 1
steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 3
P, n, dims = 8, 111059956 // scale, [128, 128, 128, 172]
cfg = R.GcnConfig(dims, epochs=100, seed=1, permute=True, overlap=True, gemm_mode=R.GEMM_TF32X3,
                  spmm_mode=R.SPMM_FAST, aggregate_input=True)
t0 = time.time()
prep = R.synth_prepare_rank(n, 28.8, 0.7, 1, dims[0], dims[-1], cfg, P, rank)
t_prep = time.time() - t0
out = {"n": n, "P": P, "rank": rank, "rows": int(prep.bounds[rank + 1] - prep.bounds[rank]), "prepare_s": round(t_prep, 1)}
out["rank_nnz"] = int(sum(prep.tile(0, rank, j)[0][-1] for j in range(P)))
import ctypes as C  # noqa: E402
for fold in (0, 2, 4):
    R.set_tuning("stage_fold", fold)
    R.set_tuning("profile", 1)
    t1 = time.time()
    g = R.Group(cfg, prep, P, local_ranks=[rank], devices=[0], transport=R.TRANSPORT_SOLO)
    t_create = time.time() - t1
    g.init_params()
    for t in range(1, 3):
        g.train_step_async(t)
    g.sync()
    g.kernels_last_step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in range(3, 3 + steps):
        g.train_step_async(t)
    g.sync()
    e1.record()
    torch.cuda.synchronize()
    a, b, c, kk = C.c_double(), C.c_double(), C.c_double(), C.c_int64()
    R._check(R.lib().mg_group_last_profile(g._h, C.byref(a), C.byref(b), C.byref(c), C.byref(kk)))
    out[f"fold{fold}"] = {"ms_per_step": e0.elapsed_time(e1) / steps, "spmm_ms": a.value / 1e3 / steps,
                          "gemm_ms": b.value / 1e3 / steps, "other_ms": c.value / 1e3 / steps,
                          "kernels_per_step": kk.value / steps, "device_bytes": int(g.buffer_audit()[2]),
                          "create_s": round(t_create, 2)}
    g.close()
    R.set_tuning("profile", 0)
# the exchange one rank receives per epoch (fp32 blocks of the other 7 ranks for every staged SpMM):
widths = [dims[0], dims[2], dims[3], dims[3], dims[2]]
out["recv_gb_per_epoch"] = (n - out["rows"]) * sum((w + 3) // 4 * 4 for w in widths) * 4 / 1e9
out["recv_ms_at_900GBs"] = out["recv_gb_per_epoch"] / 900 * 1e3
print(json.dumps(out))
