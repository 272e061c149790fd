"""Run the query hot path on one configuration (no bench bookkeeping) so ncu
can capture its kernels:  python tools/profile_query.py --config 2 --votes 1"""

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
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--nq", type=int, default=None)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--build-only", action="store_true")
ap.add_argument("--time", action="store_true", help="print ms per batched query pass")
a = ap.parse_args()
X, Q, p = workloads.generate(a.config, a.scale)
if a.nq:
    Q = Q[:a.nq]
v = a.votes or p["headline_votes"]
import time  # noqa: E402

Xd = torch.from_numpy(X).cuda()
torch.cuda.synchronize()
t0 = time.perf_counter()
index = mrpt.grow_trees(Xd, p["n_trees"], p["depth"], p["sparsity"], seed=p["seed"])
torch.cuda.synchronize()
print(f"BUILD config={a.config} n={X.shape[0]} T={p['n_trees']} depth={p['depth']} "
      f"s={time.perf_counter() - t0:.3f}")
if not a.build_only:
    D = index.device_index()
    Qd = torch.from_numpy(Q).cuda()
    if os.environ.get("MRPT_PIN"):  # route pinned for every batch size (no autotune runs under ncu)
        D.pin_route(p["k"], v, os.environ["MRPT_PIN"])
    vs = [v] if a.votes else [v]
    for _ in range(a.reps):
        ids, dists, counts = query_device(D, Qd, p["k"], v)
    torch.cuda.synchronize()
    print("mean candidates", counts.double().mean().item())
    if a.time:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            query_device(D, Qd, p["k"], v)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        ev = []
        query_device(D, Qd, p["k"], v, timer=ev)
        torch.cuda.synchronize()
        st = {}
        for name, x0, x1 in ev:
            st[name] = st.get(name, 0.0) + x0.elapsed_time(x1)
        print(f"TIME config={a.config} v={v} nq={Qd.shape[0]} ms={ms:.3f} qps={Qd.shape[0] / ms * 1e3:.0f} "
              f"stages=" + ",".join(f"{k2}:{v2:.2f}" for k2, v2 in st.items()) +
              f" variant={D.scan_choice.get((p['k'], v))}")
