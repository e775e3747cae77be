"""GPU diagnostic: full-tensor comparison of our teacher-forced step 1 with the compiled f32 reference's
step_dump (oracle/_ref, run on the box's CPU) on the products 1/16 sample, to locate where the backward
tensors diverge (which rows / entries dominate the per-column sum error).

  python scripts/step_diff_probe.py [variant ...]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

from oracle.pyoracle import Ref, make_cfg  # noqa: E402
from paper_2110_08688_b200 import rowgcn as R  # noqa: E402
import test_gpu_scale as T  # noqa: E402
from scale_common import SCALE  # noqa: E402

VARIANTS = {
    "prod": dict(gemm_mode=R.GEMM_TF32X3, spmm_mode=R.SPMM_FAST, aggregate_input=True),
    "exactgemm_fast": dict(gemm_mode=R.GEMM_EXACT, spmm_mode=R.SPMM_FAST, aggregate_input=False),
    "tc_exactspmm": dict(gemm_mode=R.GEMM_TF32X3, spmm_mode=R.SPMM_EXACT, aggregate_input=False),
}


def main():
    name = "c4s16"
    dims = SCALE[name]["dims"]
    n = SCALE[name]["n"]
    ref = Ref()
    ref.set_spmm_threads(os.cpu_count() or 8)
    c = SCALE[name]
    ds = ref.synth(c["n"], c["deg"], 0.7, 1, dims[0], dims[-1])
    d = ref.step_dump(ds, make_cfg(dims, seed=1, permute=True), 1)
    rt = {f"fwd{l}": np.asarray(d["ahw_fwd"][l]).reshape(n, -1) for l in range(3)}
    rt["loss_grad"] = np.asarray(d["loss_grad"]).reshape(n, -1)
    rt.update({f"bwd{l}": np.asarray(d["ahw_bwd"][l]).reshape(n, -1) for l in range(2)})
    print("ref loss", d["loss"], flush=True)
    for v in sys.argv[1:] or list(VARIANTS):
        T.MODES["probe"] = VARIANTS[v]
        ours = T.teacher_forced_dump(name, "probe", 1)
        for key in ["fwd0", "fwd1", "fwd2", "loss_grad", "bwd0", "bwd1"]:
            a = ours[key][:, :rt[key].shape[1]].astype(np.float64)
            b = rt[key].astype(np.float64)
            diff = a - b
            colerr = np.abs(diff.sum(0)) / np.maximum(np.abs(b).sum(0), 1e-30)
            j = int(np.argmax(colerr))
            col = diff[:, j]
            top = np.argsort(-np.abs(col))[:8]
            # sign agreement of the entries (relu masks)
            zero_a, zero_b = (a == 0), (b == 0)
            info = dict(variant=v, key=key, normwise=float(np.max(np.abs(diff)) / np.max(np.abs(b))),
                        colerr_max=float(colerr[j]), col=j, mask_flips=int(np.sum(zero_a != zero_b)),
                        nz_ours=int(np.sum(~zero_a)), nz_ref=int(np.sum(~zero_b)),
                        col_abs_sum=float(np.abs(b[:, j]).sum()), col_diff_sum=float(col.sum()),
                        top=[(int(r), float(a[r, j]), float(b[r, j])) for r in top])
            if key.startswith("bwd"):
                l = int(key[3:])
                fa = ours[f"fwd{l}"][:, :b.shape[1]]
                fb = rt[f"fwd{l}"]
                info["fwd_sign_flips"] = int(np.sum((fa > 0) != (fb > 0)))
                info["top_fwd"] = [(float(fa[r, j]), float(fb[r, j])) for r in top]
            print(json.dumps(info), flush=True)


if __name__ == "__main__":
    main()
