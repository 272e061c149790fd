"""Per-stage DRAM traffic of one batched query pass, from an ncu metrics CSV.

Capture (on the GPU box):
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none --csv --log-file gpurun_out/traffic.csv \
      python tools/profile_query.py --config 2 --votes 1 --reps 1
Summarise:
  python tools/stage_traffic.py gpurun_out/traffic.csv profiles/traffic_config2_v1.json

The query pass (from the first k_query_route launch on; run the tool with
--reps 1) is split into the bench's stages: route (k_query_route), vote
(k_vote*), scan_topk (everything after a vote: query quantisation, the
filter, exact fallback and re-rank kernels).  A large batch runs in query
chunks (one route / vote / scan per chunk): the output holds per-stage
totals of the pass (= one bench step), the per-launch means bench.py's
roofline.traffic reads ("<stage>_per_launch") and "stage_bytes_per_step"
(vote + scan)."""

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
last = seq[starts[0]:]
stages = {"route": [], "vote": [], "scan_topk": []}
seen_vote = False
for l in last:
    if "k_query_route" in l["name"]:
        stages["route"].append(l)
    elif "k_vote" in l["name"]:
        stages["vote"].append(l)
        seen_vote = True
    elif seen_vote and ("mrpt::" in l["name"] or "tc::" in l["name"]):
        stages["scan_topk"].append(l)  # (torch kernels of the calling tool are not the path)
out = {"source": src, "unit": "DRAM bytes (read + write) per stage call of the last query pass",
       "kernels": {}}
for st, ls in stages.items():
    out[st] = sum(l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0) for l in ls)
    out["kernels"][st] = [[l["name"][:70], l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0),
                           l.get("gpu__time_duration.sum", 0)] for l in ls]
for st, ls in stages.items():
    calls = sum(1 for l in ls if ("k_query_route" in l["name"] if st == "route" else
                                  "k_vote" in l["name"] if st == "vote" else
                                  "filter" in l["name"] or "k_scan_topk" in l["name"]))
    out[st + "_launches"] = calls
    out[st + "_per_launch"] = out[st] / max(1, calls)
out["stage_bytes_per_step"] = out["vote"] + out["scan_topk"]
tcf = [l for l in stages["scan_topk"] if "k_tc_filter" in l["name"]]
if tcf:  # the fused filter kernel alone (bench roofline.traffic of the tc route)
    out["k_tc_filter"] = sum(l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0) for l in tcf)
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "kernels"}, indent=1))
