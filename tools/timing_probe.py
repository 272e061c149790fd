"""Compare step timing disciplines on one configuration: contiguous events,
per-step events, per-step events with an L2 flush between steps, and the GPU
idle gap inside a step (step time minus the sum of its stage events).
usage: python tools/timing_probe.py --config 2 --votes 1"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1509_06957_b200 as mrpt  # noqa: E402
from paper_1509_06957_b200 import workloads  # noqa: E402
from paper_1509_06957_b200.search import query_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--votes", type=int, default=None)
ap.add_argument("--steps", type=int, default=10)
a = ap.parse_args()
X, Q, p = workloads.generate(a.config)
v = a.votes or p["headline_votes"]
Xd = torch.from_numpy(X).cuda()
index = mrpt.grow_trees(Xd, p["n_trees"], p["depth"], p["sparsity"], seed=p["seed"])
D = index.device_index()
Qd = torch.from_numpy(Q).cuda()
k = p["k"]
for _ in range(3):
    query_device(D, Qd, k, v)
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def run(mode):
    pairs, stages = [], []
    s, e = ev(), ev()
    torch.cuda.synchronize()
    s.record()
    for _ in range(a.steps):
        if mode in ("flush", "flush_sync"):
            flush.fill_(1)
        if mode == "flush_sync":
            torch.cuda.synchronize()
        s0, s1 = ev(), ev()
        s0.record()
        st = []
        query_device(D, Qd, k, v, timer=st)
        s1.record()
        pairs.append((s0, s1))
        stages.append(st)
    e.record()
    torch.cuda.synchronize()
    step = sum(x.elapsed_time(y) for x, y in pairs) / a.steps
    stg = sum(x.elapsed_time(y) for st in stages for _, x, y in st) / a.steps
    tot = s.elapsed_time(e) / a.steps
    print(f"{mode:12s} contiguous={tot:.3f} per_step={step:.3f} stages={stg:.3f} "
          f"gap={step - stg:.3f} ms", flush=True)


for mode in ("plain", "plain", "flush", "flush_sync", "plain"):
    run(mode)
