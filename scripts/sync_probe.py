"""Per-step cost of the synchronous C-ABI step (loss read back every step) against back-to-back async steps,
same group, same process (C4 production configuration): where the e2e number loses to the device number."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2110_08688_b200 import rowgcn as R  # noqa: E402

n, deg, dims = 2449029, 50.6, [100, 256, 256, 47]
ds = R.synth_graph(n, deg, 0.7, 1, dims[0], dims[-1])
cfg = R.GcnConfig(dims, epochs=100, seed=1, permute=True, gemm_mode=R.GEMM_TF32X3, spmm_mode=R.SPMM_FAST,
                  aggregate_input=True)
prep = R.prepare_data(ds, cfg, 1)
with R.Group(cfg, prep, 1, devices=[0]) as g:
    g.init_params()
    t = 1
    for _ in range(3):
        g.train_step(t); t += 1
    for rep in range(3):
        torch.cuda.synchronize()
        a = time.perf_counter()
        for _ in range(10):
            g.train_step_async(t); t += 1
        g.sync()
        b = time.perf_counter()
        for _ in range(10):
            g.train_step(t); t += 1
        c = time.perf_counter()
        print(f"async {1e3 * (b - a) / 10:.2f} ms/step, sync {1e3 * (c - b) / 10:.2f} ms/step", flush=True)
