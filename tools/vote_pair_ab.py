"""A/B of the list-vote kernels on one configuration, in one process: the
streamed vote (mrpt_vote_stream, one piece per id tile) against the paired
vote (mrpt_vote_pair, two tiles per 32-byte load, second parked in TMEM;
"pairw" = the same with wide counters).
Queries in the batch order the product uses (tree-0 leaf).  Candidate counts
and sorted candidate sets must be identical; prints CUDA-event times.

    python tools/vote_pair_ab.py [--config 5] [--scale 1.0] [--nq 20000] [--reps 3]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1509_06957_b200 as mrpt  # noqa: E402
from paper_1509_06957_b200 import _native, workloads  # noqa: E402
from paper_1509_06957_b200.search import _route_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--nq", type=int, default=20000)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--votes", type=int, default=None)
ap.add_argument("--variants", default="stream,pair")
args = ap.parse_args()

X, Q, p = workloads.generate(args.config, args.scale)
v = args.votes or p["headline_votes"]
Xd = torch.from_numpy(X).cuda()
index = mrpt.grow_trees(Xd, p["n_trees"], p["depth"], p["sparsity"], seed=p["seed"])
D = index.device_index()
Qd = torch.from_numpy(Q[:args.nq]).cuda()
nq = Qd.shape[0]
leaves = _route_device(Qd, D)
leaves = leaves[torch.argsort(leaves[:, 0].long(), stable=True)].contiguous()
cap = D.cap(v)
chunk = max(1, min(nq, (1 << 30) // (4 * cap)))
sizes = D.offsets[:, 1:] - D.offsets[:, :-1]
touched = float(sizes.gather(1, leaves.long().t()).sum().item())
res, ref = {}, None
for name in args.variants.split(","):
    # pairw: the paired vote with wide (10/16-bit) counters instead of the
    # saturating 8-bit ones (MRPT_VOTE_SAT=0; the layout is rebuilt)
    # pair8: plain 8-bit counters whatever T (timing only: the counts may wrap)
    sat = "0" if name == "pairw" else "1"
    mc = 255 if name == "pair8" else p["n_trees"]
    if name.startswith("pair") and (os.environ.get("MRPT_VOTE_SAT", "1") != sat or D.max_count != mc):
        os.environ["MRPT_VOTE_SAT"] = sat
        D.max_count = mc
        D._vpair = False
        torch.cuda.empty_cache()
    fn = "mrpt_vote_pair" if name.startswith("pair") else "mrpt_vote_stream"
    buf, stride, dr, base = D.vote_pair() if name.startswith("pair") else D.vote_stream()
    cand = torch.empty((nq, cap), dtype=torch.int32, device="cuda") if nq * cap * 4 < (8 << 30) else None
    cbuf = torch.empty((chunk, cap), dtype=torch.int32, device="cuda")
    counts = torch.empty(nq, dtype=torch.int32, device="cuda")

    def run(keep=False):
        for s in range(0, nq, chunk):
            e = min(nq, s + chunk)
            out = cand[s:e] if (keep and cand is not None) else cbuf
            _native.call(fn, _native.ptr(buf), int(stride), _native.ptr(dr), _native.ptr(base), D.n, D.T,
                         D.depth, int(D.max_count), _native.ptr(leaves[s:e]), e - s, int(v), _native.ptr(out),
                         int(cap), _native.ptr(counts[s:e]), _native.stream_ptr())

    run(keep=True)
    torch.cuda.synchronize()
    # canonical form: each query's listed ids sorted (order within a tile is not kept)
    digest = int(counts.sum().item())
    if cand is not None:
        m = counts.clamp(max=cap).long()
        ar = torch.arange(cap, device="cuda")[None, :]
        canon = torch.where(ar < m[:, None], cand, torch.full_like(cand, 2**31 - 1)).sort(dim=1).values
        digest = (digest, int((canon.long() * 2654435761 % 1000000007).sum().item()))
    ts = []
    for _ in range(args.reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    c = counts.cpu().numpy()
    if ref is None:
        ref = (c, digest)
    res[name] = {"layout_gb": round(buf.numel() * 4 / 1e9, 2), "ms": round(ms, 3),
                 "ms_per_100k": round(ms * 1e5 / nq, 2), "leaf_id_gbs": round(4 * touched / (ms / 1e3) / 1e9, 1),
                 "same_counts": bool(np.array_equal(c, ref[0])), "same_sets": digest == ref[1],
                 "sat": mrpt.search.vote_stats(reset=True)}
    del cand
print(json.dumps({"config": args.config, "scale": args.scale, "nq": nq, "v": v,
                  "leaf_id_bytes_per_query": 4 * touched / nq, **res}))
