"""Per-kernel summary of an ncu launch list taken with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,
sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --csv:
launches, serialised ms, share, DRAM GB, DRAM GB/s, time-weighted FP64-pipe %.
usage: python tools/build_launch_summary.py launches.csv"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
per = defaultdict(dict)
for r in rows[hdr + 1:]:
    if len(r) > vi and r[vi]:
        per[(r[ii], r[ki].split("(")[0].replace("void ", ""))][r[mi]] = (float(r[vi].replace(",", "")), r[ui])
tscale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
bscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for (_, k), m in per.items():
    t, u = m["gpu__time_duration.sum"]
    t *= tscale[u]
    a = agg[k]
    a[0] += 1
    a[1] += t
    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        if key in m:
            a[2] += m[key][0] * bscale[m[key][1]]
    a[3] += m.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", (0.0, ""))[0] * t
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':32s} {'launches':>8s} {'ms':>9s} {'share':>6s} {'DRAM GB':>8s} {'GB/s':>7s} {'fp64 %':>6s}")
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:32]:32s} {a[0]:8d} {a[1] / 1e3:9.3f} {100 * a[1] / tot:5.1f}% {a[2] / 1e9:8.3f} "
          f"{a[2] / (a[1] * 1e-6) / 1e9 if a[1] else 0:7.0f} {a[3] / a[1] if a[1] else 0:6.1f}")
print(f"{'TOTAL':32s} {sum(a[0] for a in agg.values()):8d} {tot / 1e3:9.3f}")
