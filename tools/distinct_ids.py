"""Distinct ids per query among its T leaves (the candidate count at v=1) and
at a few thresholds: sizes the counter structures of the vote.
usage: python tools/distinct_ids.py [config] [nq]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1509_06957_b200 as mrpt  # noqa: E402
from paper_1509_06957_b200 import workloads  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 200
X, Q, p = workloads.generate(cfg)
index = mrpt.grow_trees(torch.from_numpy(X).cuda(), p["n_trees"], p["depth"], p["sparsity"], seed=p["seed"])
for v in (1, 2, 3, 5, 10):
    _, _, counts = mrpt.approximate_knn_batch(Q[:nq], p["k"], index, v)
    c = counts.astype(np.int64)
    print(f"config {cfg} v={v}: candidates mean {c.mean():.0f} max {c.max()} (n={X.shape[0]}, "
          f"T={p['n_trees']}, occurrences/query ~{p['n_trees'] * X.shape[0] / 2 ** p['depth']:.0f})", flush=True)
