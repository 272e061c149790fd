"""Print the tc-route kernels of an ncu launch list in order (us)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
keys = ("tc", "tiled", "rerank", "vote", "quantize_q8", "route")
for r in rows[hdr + 1:]:
    if len(r) > vi and any(k in r[ki] for k in keys):
        print(f"{r[ki].split('(')[0][:40]:40s} {float(r[vi].replace(',', '')) / 1000:9.1f}")
