"""Small end-to-end runs for compute-sanitizer: exact and FAST/TF32X3 training at P = 1 and 2 (in-process),
the device partitioner, bench-spmm and a kernel-level SpMM with hub segments."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402,F401
from paper_2110_08688_b200 import rowgcn as R  # noqa: E402

R.set_tuning("heavy_row", 64)  # hub segments + hub-row kernels on a small graph
ds = R.synth_graph(3000, 12.0, 0.7, 2, 40, 5)
for gm, sm in [(R.GEMM_EXACT, R.SPMM_EXACT), (R.GEMM_TF32X3, R.SPMM_FAST)]:
    for P in (1, 2):
        cfg = R.GcnConfig([40, 64, 5], epochs=2, seed=1, permute=True, overlap=P > 1, gemm_mode=gm, spmm_mode=sm)
        art = R.train_run(ds, cfg, R.TrainOptions(workers=P, devices=[0] * P,
                                                  transport=R.TRANSPORT_NCCL if P == 1 else R.TRANSPORT_LOCAL))
        print("train", gm, sm, P, art.epoch_loss, flush=True)
# products-like widths: 256-column tiles, N = 48 tiles, 32-row TN stages with TMEM drains, half-warp softmax
ds2 = R.synth_graph(3000, 12.0, 0.7, 3, 100, 47)
cfg = R.GcnConfig([100, 256, 256, 47], epochs=2, seed=1, permute=True)
print("train c4-like", R.train_run(ds2, cfg, R.TrainOptions()).epoch_loss, flush=True)
with R.Group(cfg, R.prepare_data(ds2, cfg, 1), 1, devices=[0]) as g:  # backward from a written gradient
    g.init_params()
    g.forward()
    g.backward()
    print("backward", float(abs(g.read(R.T_WGRAD, 1)).sum()) >= 0, flush=True)
cfg = R.GcnConfig([40, 64, 5], epochs=1, seed=1, permute=True)
R.prepare_data(ds, cfg, 2, device=0)
print("bench_spmm", R.bench_spmm(ds, workers=2, devices=[0, 0], transport=R.TRANSPORT_LOCAL)["wall_us"] > 0)
# round 2: the fp16 GeMM split (K = 256 > gemm_f16_min_k, row maxima from the producers), aggregate_input,
# stage folding at P = 4 (in-process), the per-rank synthetic path + the solo transport
cfg = R.GcnConfig([100, 256, 256, 47], epochs=2, seed=1, permute=True, aggregate_input=True,
                  gemm_mode=R.GEMM_TF32X3, spmm_mode=R.SPMM_FAST)
R.set_tuning("gemm_f16", 1)
print("train f16 split", R.train_run(ds2, cfg, R.TrainOptions()).epoch_loss, flush=True)
R.set_tuning("gemm_f16", 0)
R.set_tuning("stage_fold", 2)
cfg = R.GcnConfig([40, 64, 5], epochs=2, seed=1, permute=True, overlap=True, aggregate_input=True,
                  gemm_mode=R.GEMM_TF32X3, spmm_mode=R.SPMM_FAST)
print("train fold", R.train_run(ds, cfg, R.TrainOptions(workers=4, devices=[0] * 4,
                                                       transport=R.TRANSPORT_LOCAL)).epoch_loss, flush=True)
R.set_tuning("stage_fold", 0)
prep = R.synth_prepare_rank(3000, 12.0, 0.7, 2, 40, 5, cfg, 4, 2)
with R.Group(cfg, prep, 4, local_ranks=[2], devices=[0], transport=R.TRANSPORT_SOLO) as g:
    g.init_params()
    print("solo", g.train_step(1) == g.train_step(1) or True, flush=True)
# late round 2: the step as a CUDA graph (default) with the opt-in Â·X cache, a feature write in between
R.set_tuning("ax_cache", 1)
cfg = R.GcnConfig([100, 256, 256, 47], epochs=3, seed=1, permute=True, aggregate_input=True,
                  gemm_mode=R.GEMM_TF32X3, spmm_mode=R.SPMM_FAST)
with R.Group(cfg, R.prepare_data(ds2, cfg, 1), 1, devices=[0]) as g:
    g.init_params()
    losses = [g.train_step(t) for t in (1, 2)]
    g.write(R.T_X, 0, g.read(R.T_X, 0) * np.float32(0.5))
    losses.append(g.train_step(3))
    print("ax_cache + graph", losses, g.graph_steps(), flush=True)
R.set_tuning("ax_cache", 0)
