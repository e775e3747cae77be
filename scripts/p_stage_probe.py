"""C4 (products-shaped) training steps at P = 2/4/8 on ONE B200 with the in-process transport: the same
per-stage tiles, work lists and kernels an NCCL run on P GPUs launches, here for all P ranks on one device.
Run under ncu (kernels serialised, profiled region = the timed steps only):

  ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \\
      --csv --log-file gpurun_out/p8.csv python scripts/p_stage_probe.py 8
  python scripts/p_stage_probe.py --summarise gpurun_out/p8.csv 8

The summary divides every kernel's total by P (ranks are balanced by the random permutation) and models the
P-GPU epoch: per layer and direction, stages overlap their feature broadcast (the stage block, rows/P x
width x 4 B, over NVLink 5 at 900 GB/s ingress) with the previous stage's SpMM (inc/dist_spmm.hpp:57-103).
"""
import csv
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

N, DEG, DIMS = 2449029, 50.6, [100, 256, 256, 47]


def run(P, steps=1, timed=0):
    """steps: steps inside the profiler range (ncu); timed > 0: instead, time `timed` back-to-back steps
    with CUDA events (no profiler) — all P ranks share the one GPU, so the step time / P estimates one
    rank's compute time on P GPUs (the in-process broadcasts are device copies). MG_TUNE="k=v,..." sets
    tuning keys."""
    import torch
    from paper_2110_08688_b200 import rowgcn as R
    for kv in filter(None, os.environ.get("MG_TUNE", "").split(",")):
        k, v = kv.split("=")
        R.set_tuning(k, int(v))
    ds = R.synth_graph(N, DEG, 0.7, 1, DIMS[0], DIMS[-1])
    cfg = R.GcnConfig(DIMS, epochs=steps, seed=1, permute=True, overlap=True, gemm_mode=R.GEMM_TF32X3,
                      spmm_mode=R.SPMM_FAST, aggregate_input=True)
    prep = R.prepare_data(ds, cfg, P, device=0)
    with R.Group(cfg, prep, P, devices=[0] * P, transport=R.TRANSPORT_LOCAL if P > 1 else R.TRANSPORT_NCCL) as g:
        g.init_params()
        g.train_step(1)
        g.sync()
        torch.cuda.synchronize()
        if timed:
            for t in range(3):
                g.train_step_async(2 + t)
            g.sync()
            torch.cuda.synchronize()
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record()
            for t in range(timed):
                g.train_step_async(5 + t)
            g.sync()
            t1.record()
            torch.cuda.synchronize()
            ms = t0.elapsed_time(t1) / timed
            print(json.dumps({"P": P, "ms_per_step_all_ranks_one_gpu": ms, "est_ms_per_rank": ms / P}))
            return
        torch.cuda.profiler.start()
        for t in range(steps):
            loss = g.train_step(2 + t)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    print(json.dumps({"P": P, "loss": loss}))


def summarise(path, P, steps=1):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    idi = h.index("ID")
    per = defaultdict(dict)
    names = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        if r[mi].startswith("dram__bytes"):
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        elif r[mi] == "gpu__time_duration.sum":
            v *= {"ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
        per[r[idi]][r[mi]] = v
        names[r[idi]] = r[ki].split("(")[0].replace("void ", "")
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in per.items():
        a = agg[names[i]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    out = {"P": P, "per_rank_ms": tot / P / steps / 1e3, "kernels": {}}
    for k, (n, us, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out["kernels"][k] = dict(launches_per_rank=n / P / steps, ms_per_rank=us / P / steps / 1e3,
                                 dram_gb_per_rank=b / P / steps / 1e9,
                                 gbs=(b / (us * 1e-6) / 1e9) if us else None)
    spmm_ms = sum(v["ms_per_rank"] for k, v in out["kernels"].items() if "spmm" in k)
    gemm_ms = sum(v["ms_per_rank"] for k, v in out["kernels"].items() if "gemm" in k or "reduce_partials" in k)
    out["spmm_ms_per_rank"], out["gemm_ms_per_rank"] = spmm_ms, gemm_ms
    # epoch model on P GPUs: the staged SpMMs of one step (aggregate_input: layer 0 forward d0 wide, no layer-0
    # backward SpMM) — each stage j > 0 waits for its broadcast; with overlap the broadcast of stage j runs
    # beside the SpMM of stage j - 1. Stage SpMM time = the measured per-rank SpMM time spread over the
    # stages in proportion to width (the same tiles at every width).
    rows_p = N / P
    widths = [DIMS[0], DIMS[2], DIMS[3], DIMS[3], DIMS[2]]  # fwd l0 (aggregated input), l1, l2; bwd l2, l1
    wsum = sum(widths)
    model = 0.0
    bw = 900e9
    for w in widths:
        st = spmm_ms * w / wsum / P  # ms per stage
        bc = rows_p * w * 4 / bw * 1e3  # ms per stage broadcast
        model += st + (P - 1) * max(st, bc) if P > 1 else st
    other = out["per_rank_ms"] - spmm_ms - gemm_ms
    out["model_epoch_ms"] = model + gemm_ms + other
    out["model_note"] = ("stages: first SpMM, then P-1 x max(SpMM stage, its broadcast at 900 GB/s ingress); "
                         "plus the rank's GeMMs and other kernels; W-grad all-reduce (~0.3 MB) ignored")
    return out


if __name__ == "__main__":
    if sys.argv[1] == "--summarise":
        print(json.dumps(summarise(sys.argv[2], int(sys.argv[3])), indent=1))
    else:
        run(int(sys.argv[1]), timed=int(sys.argv[2]) if len(sys.argv) > 2 else 0)
