"""Per-opcode and per-instruction hot spots of one kernel in an ncu report
(needs --set full / source counters).
usage: python tools/sass_hot.py report.ncu-rep kernel-regex [threshold-pct]"""
import collections
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.4
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      "regex:" + kern, "--launch-count", "1", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
ie, isamp, src = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


data = [r for r in rows[hi + 1:] if len(r) > ie and r[0] != "Address"]
tot = sum(num(r[ie]) for r in data)
ts = sum(num(r[isamp]) for r in data) or 1.0
print("total inst %.4g  samples %d  sass %d" % (tot, ts, len(data)))
op, sp = collections.Counter(), collections.Counter()
for r in data:
    o = [x for x in r[src].strip().split() if not x.startswith("@")]
    name = o[0].split(".")[0] if o else "?"
    op[name] += num(r[ie])
    sp[name] += num(r[isamp])
for k, v in op.most_common(28):
    print("%-10s %5.1f%% inst %5.1f%% samples" % (k, 100 * v / tot, 100 * sp[k] / ts))
print()
for idx, r in enumerate(data):
    if num(r[ie]) > tot * thr / 100 or num(r[isamp]) > ts * thr / 100:
        print("%4d %s %5.2f%% %5.2f%%  %s" % (idx, r[0][-5:], 100 * num(r[ie]) / tot,
                                            100 * num(r[isamp]) / ts, r[src].strip()[:96]))
