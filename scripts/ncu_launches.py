"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel totals and shares."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = defaultdict(lambda: [0, 0.0])
order = []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"].replace(",", ""))
    unit = d["Metric Unit"]
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6,
             "s": 1e6}.get(unit, 1.0)
    name = d["Kernel Name"].split("(")[0][:70]
    agg[name][0] += 1
    agg[name][1] += v * scale
    order.append((name, v * scale, d.get("Grid Size", ""), d.get("Block Size", "")))
tot = sum(v[1] for v in agg.values())
print(f"{'total_us':>12} {'n':>4} {'share':>6}  kernel")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[1]:12.1f} {v[0]:4d} {100 * v[1] / tot:5.1f}%  {k}")
print(f"{tot:12.1f} total us over {len(order)} launches")
if "-v" in sys.argv:
    for name, us, g, b in order:
        print(f"  {us:10.1f}  {g:>14} {b:>10}  {name}")
