"""Host-side enqueue time of the query path (no synchronisation inside):
if it approaches the GPU time per call, the GPU idles between launches.
usage: python tools/host_overhead.py --config 2 --votes 1"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1509_06957_b200 as mrpt  # noqa: E402
from paper_1509_06957_b200 import workloads  # noqa: E402
from paper_1509_06957_b200.search import query_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--votes", type=int, default=1)
a = ap.parse_args()
X, Q, p = workloads.generate(a.config)
index = mrpt.grow_trees(torch.from_numpy(X).cuda(), p["n_trees"], p["depth"], p["sparsity"],
                        seed=p["seed"])
D = index.device_index()
Qd = torch.from_numpy(Q).cuda()
k, v = p["k"], a.votes
for _ in range(3):
    query_device(D, Qd, k, v)
torch.cuda.synchronize()
for m in (10000, 2500, 1250):
    qb = Qd[:m]
    hs = []
    for _ in range(20):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        query_device(D, qb, k, v)
        hs.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        query_device(D, qb, k, v)
    e1.record()
    torch.cuda.synchronize()
    print(f"nq={m}: host enqueue {1e3 * np.median(hs):.3f} ms, gpu {e0.elapsed_time(e1) / 20:.3f} ms per call",
          flush=True)
Qpin = torch.from_numpy(Q).pin_memory()
for _ in range(3):
    mrpt.approximate_knn_batch(Qpin, k, index, v)
ts = []
for _ in range(10):
    t0 = time.perf_counter()
    mrpt.approximate_knn_batch(Qpin, k, index, v)
    ts.append(time.perf_counter() - t0)
print(f"e2e approximate_knn_batch (pinned 10k): {1e3 * np.median(ts):.3f} ms", flush=True)
