"""Query-order A/B at one configuration: stage times of the batched query
pass (CUDA events) under different batch orders (search._order_hook).
usage: python tools/order_ab.py [config] [scale]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1509_06957_b200 as mrpt  # noqa: E402
from paper_1509_06957_b200 import search, workloads  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
X, Q, p = workloads.generate(cfg, scale)
index = mrpt.grow_trees(torch.from_numpy(X).cuda(), p["n_trees"], p["depth"], p["sparsity"], seed=0)
D = index.device_index()
Qd = torch.from_numpy(Q).cuda()
k, v = p["k"], p["headline_votes"]
L = 1 << p["depth"]
rng = np.random.default_rng(0)
centres = torch.from_numpy((3.0 * rng.standard_normal((1024, X.shape[1]))).astype(np.float32)).cuda()


def by_cluster(leaves, Qd):
    lab = torch.cdist(Qd, centres).argmin(1)
    return torch.argsort(lab * L + leaves[:, 0].long(), stable=True).int()


def kmeans_order(K, iters):
    def f(leaves, Qd):
        g = torch.Generator(device="cuda").manual_seed(1)
        C = Qd[torch.randperm(Qd.shape[0], device="cuda", generator=g)[:K]].clone()
        for _ in range(iters):
            lab = torch.cdist(Qd, C).argmin(1)
            C.index_add_(0, lab, Qd)  # running mean: old centre counts as one member
            cnt = torch.bincount(lab, minlength=K).float() + 1
            C /= cnt[:, None]
        lab = torch.cdist(Qd, C).argmin(1)
        return torch.argsort(lab * L + leaves[:, 0].long(), stable=True).int()
    return f


ref = None
for name, hook in (("tree-0 leaf", None), ("true cluster", by_cluster), ("kmeans K=1000 x3", kmeans_order(1000, 3)),
                   ("kmeans K=300 x3", kmeans_order(300, 3)), ("kmeans K=3000 x2", kmeans_order(3000, 2))):
    search._order_hook = hook
    best = None
    for rep in range(3):
        timer = []
        out = search.query_device(D, Qd, k, v, timer=timer)
        torch.cuda.synchronize()
        st = {}
        for nm, a, b in timer:
            st[nm] = st.get(nm, 0.0) + a.elapsed_time(b)
        if rep and (best is None or sum(st.values()) < sum(best.values())):
            best = st
    sig = tuple(t.cpu().numpy().tobytes() for t in out)
    same = ref is None or sig == ref
    ref = ref or sig
    print(f"{name:20s} " + " ".join(f"{a}={b:.1f}" for a, b in best.items()) + f" total={sum(best.values()):.1f} same={same}",
          flush=True)
