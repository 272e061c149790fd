"""A/B of the K3 vote kernels on one configuration, in one process: the
streamed vote (mrpt_vote_stream) against the directory vote (mrpt_vote with
the u16 tile directory).  Same candidate counts required; prints per-kernel
CUDA-event times and the algorithmic leaf-id rate.

    python tools/vote_ab.py [--config 5] [--scale 1.0] [--nq 20000] [--reps 3]
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
args = ap.parse_args()

X, Q, p = workloads.generate(args.config, args.scale)
v = args.votes or p["headline_votes"]
Xd = torch.from_numpy(X).cuda()
index = mrpt.grow_trees(Xd, p["n_trees"], p["depth"], p["sparsity"], seed=p["seed"])
D = index.device_index()
Qd = torch.from_numpy(Q[:args.nq]).cuda()
nq = Qd.shape[0]
leaves = _route_device(Qd, D)
cap = D.cap(v)
chunk = max(1, min(nq, (1 << 30) // (4 * cap)))
sizes = D.offsets[:, 1:] - D.offsets[:, :-1]
touched = float(sizes.gather(1, leaves.long().t()).sum().item())
res = {}
for name in ("stream", "dir"):
    cand = torch.empty((chunk, cap), dtype=torch.int32, device="cuda")
    counts = torch.empty(nq, dtype=torch.int32, device="cuda")

    def run():
        for s in range(0, nq, chunk):
            e = min(nq, s + chunk)
            if name == "stream":
                qs, tstride, qdir, qbase = D.vote_stream()
                _native.call("mrpt_vote_stream", _native.ptr(qs), int(tstride), _native.ptr(qdir),
                             _native.ptr(qbase), D.n, D.T, D.depth, int(D.max_count),
                             _native.ptr(leaves[s:e]), e - s, int(v), _native.ptr(cand), int(cap),
                             _native.ptr(counts[s:e]), _native.stream_ptr())
            else:
                _native.call("mrpt_vote", _native.ptr(D.indices), _native.ptr(D.offsets), D.n, D.T,
                             D.depth, _native.ptr(leaves[s:e]), e - s, int(v), int(D.leaves_sorted),
                             int(D.max_count), _native.ptr(D.vote_dir()), _native.ptr(cand), int(cap),
                             _native.ptr(counts[s:e]), _native.stream_ptr())

    run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    res[name] = {"ms": ms, "gbs": 4 * touched / (ms / 1e3) / 1e9, "counts_sum": int(counts.sum().item()),
                 "ms_per_100k": ms * 1e5 / nq}
    res[name + "_counts"] = counts.cpu().numpy()
same = bool(np.array_equal(res.pop("stream_counts"), res.pop("dir_counts")))
print(json.dumps({"config": args.config, "scale": args.scale, "nq": nq, "v": v, "same_counts": same,
                  "leaf_id_bytes_per_query": 4 * touched / nq, **res}))
