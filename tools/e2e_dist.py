"""Per-call wall time distribution of the e2e path (config 2, pinned host
queries): finds stalls that a mean over a few calls would hide."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1509_06957_b200 as mrpt  # noqa: E402
from paper_1509_06957_b200 import workloads  # noqa: E402
from paper_1509_06957_b200.search import query_device  # noqa: E402

X, Q, p = workloads.generate(2)
Xd = torch.from_numpy(X).cuda()
index = mrpt.grow_trees(Xd, p["n_trees"], p["depth"], p["sparsity"], seed=0)
D = index.device_index()
Qd = torch.from_numpy(Q).cuda()
for _ in range(4):
    query_device(D, Qd, p["k"], 1)
torch.cuda.synchronize()
Qp = torch.from_numpy(Q).pin_memory()
ts = []
for i in range(60):
    t = time.perf_counter()
    mrpt.approximate_knn_batch(Qp, p["k"], index, 1)
    ts.append((time.perf_counter() - t) * 1e3)
ts = np.array(ts)
print("first 12 calls ms:", np.round(ts[:12], 2).tolist())
print("median %.3f  mean(10..59) %.3f  max %.3f  p90 %.3f" % (np.median(ts), ts[10:].mean(), ts.max(),
                                                            np.percentile(ts, 90)))
print("choice:", D.scan_choice_by_size)
