"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel launch count, total time and share.  usage: launch_summary.py file.csv"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
mi = h.index("Metric Name") if "Metric Name" in h else None
agg = defaultdict(lambda: [0, 0.0])
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
         "second": 1e6, "s": 1e6}
for r in rows[hdr + 1:]:
    if len(r) <= vi or not r[vi]:
        continue
    if mi is not None and r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].replace("void ", "")
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':44s} {'launches':>8s} {'total ms':>10s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:44]:44s} {v[0]:8d} {v[1] / 1e3:10.2f} {100 * v[1] / tot:5.1f}%")
print(f"{'TOTAL':44s} {sum(v[0] for v in agg.values()):8d} {tot / 1e3:10.2f}")
