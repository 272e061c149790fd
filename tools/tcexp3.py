"""e2e and device timing of config 2 through the public API (tc route pinned)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1509_06957_b200 as mrpt  # noqa: E402
from paper_1509_06957_b200 import workloads  # noqa: E402

X, Q, p = workloads.generate(2)
index = mrpt.grow_trees(X, p["n_trees"], p["depth"], sparsity=p["sparsity"], seed=0)
Qp = torch.from_numpy(Q).pin_memory()
for nq in (1250, 2917, 8750, 10000):
    for _ in range(3):
        ids, d, c = mrpt.approximate_knn_batch(Qp[:nq], p["k"], index, 1)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        ids, d, c = mrpt.approximate_knn_batch(Qp[:nq], p["k"], index, 1)
    dt = (time.perf_counter() - t) / 5
    print(f"nq={nq} e2e {dt * 1e3:.3f} ms  {nq / dt:.0f} qps  route={index.device_index().scan_choice}", flush=True)
