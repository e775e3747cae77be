"""From an ncu --set full capture of one training step, write profiles/spmm_traffic.json: the SpMM
kernels' measured DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per staged-SpMM launch, for
bench.py's roofline.traffic.
    python scripts/spmm_traffic.py gpurun_out/rNN_full.ncu-rep|raw.csv c4 5 [note]"""
import csv
import io
import json
import os
import subprocess
import sys

rep, cfg, launches = sys.argv[1], sys.argv[2], int(sys.argv[3])
note = sys.argv[4] if len(sys.argv) > 4 else ""
out = (open(rep).read() if rep.endswith(".csv") else
       subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
total, kernels = 0.0, 0
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    if "spmm" not in name:
        continue
    kernels += 1
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(m)
        v = float(r[i].replace(",", "")) * scale[units[i]]
        total += 0.0 if v != v else v  # ncu reports -nan for some ~80 us hub-reduction launches (MB-scale)
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path = os.path.join(root, "profiles", "spmm_traffic.json")
data = json.load(open(path)) if os.path.exists(path) else {}
data[cfg] = {"dram_bytes_per_launch": total / launches, "dram_bytes_per_step": total, "spmm_kernels": kernels,
             "launches_per_step": launches, "source": os.path.basename(rep), "note": note}
json.dump(data, open(path, "w"), indent=1)
print(json.dumps(data[cfg]))
