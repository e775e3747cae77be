"""Phase timings of the end-to-end path (group create / init / K synchronous steps / W read-back)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MGGCN_TIMING", "1")
from paper_2110_08688_b200 import rowgcn as R  # noqa: E402

SHAPES = {"c4": (2449029, 50.6, [100, 256, 256, 47]), "c2": (169343, 13.6, [128, 256, 256, 40]),
          "c1": (2708, 3.9, [1433, 16, 7])}
for kv in filter(None, os.environ.get("MG_TUNE", "").split(",")):  # e.g. MG_TUNE=step_graph=0
    k, v = kv.split("=")
    R.set_tuning(k, int(v))
n, deg, dims = SHAPES[sys.argv[1] if len(sys.argv) > 1 else "c4"]
t0 = time.time()
ds = R.synth_graph(n, deg, 0.7, 1, dims[0], dims[-1])
t1 = time.time()
cfg = R.GcnConfig(dims, epochs=10, seed=1, permute=True, gemm_mode=R.GEMM_TF32X3, spmm_mode=R.SPMM_FAST,
                  aggregate_input=True)  # the bench configuration
prep = R.prepare_data(ds, cfg, 1)
t2 = time.time()
print(f"synth {t1 - t0:.2f} s, prepare {t2 - t1:.2f} s", flush=True)
for rep in range(int(os.environ.get("REPS", "2"))):
    a = time.time()
    g = R.Group(cfg, prep, 1, devices=[0])
    b = time.time()
    g.init_params()
    c = time.time()
    st = []
    for t in range(1, 11):
        s0 = time.time()
        g.train_step(t)
        st.append(1e3 * (time.time() - s0))
    d = time.time()
    ws = g.params(0)
    e = time.time()
    g.close()
    f = time.time()
    print(f"create {1e3 * (b - a):.1f} ms, init {1e3 * (c - b):.1f} ms, 10 steps {1e3 * (d - c):.1f} ms, "
          f"params {1e3 * (e - d):.1f} ms, close {1e3 * (f - e):.1f} ms; steps " + " ".join(f"{x:.1f}" for x in st),
          flush=True)
