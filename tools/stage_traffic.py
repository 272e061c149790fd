"""Per-stage DRAM traffic of one batched query pass, from an ncu metrics CSV.

Capture (on the GPU box):
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none --csv --log-file gpurun_out/traffic.csv \
      python tools/profile_query.py --config 2 --votes 1 --reps 1
Summarise:
  python tools/stage_traffic.py gpurun_out/traffic.csv profiles/traffic_config2_v1.json

The last query pass (from the last k_query_route launch on) is split into the
bench's stages: route (k_query_route), vote (k_vote*), scan_topk (everything
after the vote: query quantisation, the cuBLASLt GEMM, the filter, exact
fallback and re-rank kernels).  Bytes are per stage call, i.e. per batch of
queries, as bench.py's roofline.traffic expects."""

import csv
import json
import sys

src, dst = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(src)))
hi = [i for i, r in enumerate(rows) if r and "Kernel Name" in r][0]
h = rows[hi]
kn, mn, mv, mu, iid = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
launches = {}
order = []
for r in rows[hi + 1:]:
    if len(r) <= mv:
        continue
    key = r[iid]
    if key not in launches:
        launches[key] = {"name": r[kn]}
        order.append(key)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "usecond": 1e3,
             "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(r[mu], 1)
    launches[key][r[mn]] = float(r[mv].replace(",", "")) * scale
seq = [launches[k] for k in order]
starts = [i for i, l in enumerate(seq) if "k_query_route" in l["name"]]
last = seq[starts[-1]:]
stages = {"route": [], "vote": [], "scan_topk": []}
seen_vote = False
for l in last:
    if "k_query_route" in l["name"]:
        stages["route"].append(l)
    elif "k_vote" in l["name"]:
        stages["vote"].append(l)
        seen_vote = True
    elif seen_vote and ("mrpt::" in l["name"] or "tc::" in l["name"] or "cutlass" in l["name"]
                        or "gemm" in l["name"]):
        stages["scan_topk"].append(l)  # (torch kernels of the calling tool are not the path)
out = {"source": src, "unit": "DRAM bytes (read + write) per stage call of the last query pass",
       "kernels": {}}
for st, ls in stages.items():
    out[st] = sum(l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0) for l in ls)
    out["kernels"][st] = [[l["name"][:70], l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0),
                           l.get("gpu__time_duration.sum", 0)] for l in ls]
tcf = [l for l in stages["scan_topk"] if "k_tc_filter" in l["name"]]
if tcf:  # the fused filter kernel alone (bench roofline.traffic of the tc route)
    out["k_tc_filter"] = sum(l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0) for l in tcf)
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "kernels"}, indent=1))
