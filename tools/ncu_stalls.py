"""Per-SASS-line stall samples of one kernel from an ncu report (source page):
the lines holding most samples, with their dominant stall reasons.
usage: python tools/ncu_stalls.py report.ncu-rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
h = rows[1]
si, wi, ei = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
data = rows[2:]
tot = sum(int(r[wi] or 0) for r in data)
print(f"samples {tot}")
for i, r in sorted(enumerate(data), key=lambda x: -int(x[1][wi] or 0))[:top]:
    w = int(r[wi] or 0)
    rs = sorted(((int(r[h.index(c)] or 0), c[6:]) for c in reasons), reverse=True)[:3]
    print(f"{i:4d} {100 * w / tot:5.1f}%  exec={r[ei]:>10s}  {r[si].strip()[:55]:55s} "
          + " ".join(f"{n}:{v}" for v, n in rs if v))
