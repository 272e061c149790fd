"""e2e (pinned host queries in, host results out) of config 2 for several
pipelining schedules (MRPT_PIPE)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1509_06957_b200 as mrpt  # noqa: E402
from paper_1509_06957_b200 import workloads  # noqa: E402

X, Q, p = workloads.generate(2)
index = mrpt.grow_trees(X, p["n_trees"], p["depth"], sparsity=p["sparsity"], seed=0)
Qp = torch.from_numpy(Q).pin_memory()
for mode in ("p2", "p4", "p6", "p8"):
    os.environ["MRPT_PIPE_PIECES"] = mode[1:]
    for _ in range(3):
        mrpt.approximate_knn_batch(Qp, p["k"], index, 1)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10):
        mrpt.approximate_knn_batch(Qp, p["k"], index, 1)
    dt = (time.perf_counter() - t) / 10
    print(f"mode={mode or 'default'} e2e {dt * 1e3:.3f} ms {Q.shape[0] / dt:.0f} qps", flush=True)
# raw H2D of the queries
d = torch.empty(Q.shape, dtype=torch.float32, device="cuda")
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10):
    d.copy_(Qp, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D {Q.nbytes / 1e6:.1f} MB: {(time.perf_counter() - t) / 10 * 1e3:.3f} ms")
