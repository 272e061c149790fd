"""How many leaf slices do queries that run at the same time share?  Builds a
configuration, routes its queries, and for several query orders reports
 - the fraction of trees in which consecutive queries reach the same leaf,
 - distinct (tree, leaf) slices per block of B consecutive queries / (B*T)
   (1.0 = no sharing; the streamed vote reads each block's slices about once
   from DRAM when the block runs concurrently).
usage: python tools/leaf_sharing.py [config] [scale] [B]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1509_06957_b200 as mrpt  # noqa: E402
from paper_1509_06957_b200 import workloads  # noqa: E402
from paper_1509_06957_b200.search import _route_device  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
B = int(sys.argv[3]) if len(sys.argv) > 3 else 148
X, Q, p = workloads.generate(cfg, scale)
index = mrpt.grow_trees(torch.from_numpy(X).cuda(), p["n_trees"], p["depth"], p["sparsity"], seed=0)
D = index.device_index()
Qd = torch.from_numpy(Q).cuda()
leaves = _route_device(Qd, D).long()  # (nq, T)
nq, T = leaves.shape
L = 1 << p["depth"]
keys = leaves + torch.arange(T, device=leaves.device)[None, :] * L


def report(name, order):
    lp = leaves[order]
    kp = keys[order]
    same = (lp[1:] == lp[:-1]).float().mean().item()
    fr = []
    for b0 in range(0, nq - B + 1, B * 8):  # every 8th block
        fr.append(torch.unique(kp[b0:b0 + B]).numel() / (B * T))
    print(f"{name:34s} consecutive-same {same:.3f}  distinct/(B*T) at B={B}: {np.mean(fr):.3f}", flush=True)


ar = torch.arange(nq, device=leaves.device)
report("original order", ar)
report("tree-0 leaf", torch.argsort(leaves[:, 0], stable=True))
o = ar
for t in (1, 0):
    o = o[torch.argsort(leaves[o, t], stable=True)]
report("tree-0 then tree-1 leaf", o)
# leaf prefix orders: top h levels of several trees concatenated (coarse cells)
for h, nt in ((3, 4), (4, 3), (6, 2), (2, 6), (1, 12), (1, 16), (2, 8)):
    sig = torch.zeros(nq, dtype=torch.long, device=leaves.device)
    for t in range(nt):
        sig = (sig << h) | (leaves[:, t] >> (p["depth"] - h))
    o = torch.argsort(sig * L + leaves[:, 0], stable=True)
    report(f"top {h} levels of {nt} trees, then leaf0", o)
if cfg == 5:
    rng = np.random.default_rng(0)
    centres = torch.from_numpy((3.0 * rng.standard_normal((1024, X.shape[1]))).astype(np.float32)).cuda()
    lab = torch.cdist(Qd, centres).argmin(1)
    report("true cluster, then leaf0", torch.argsort(lab * L + leaves[:, 0], stable=True))
    # greedy chain within the batch by Euclidean nearest unvisited neighbour is too slow; instead
    # order by the nearest data-independent random hyperplane cells
    R = torch.randn(X.shape[1], 20, device=Qd.device)
    bits = ((Qd - Qd.mean(0)) @ R > 0).long()
    sig = (bits * (1 << torch.arange(20, device=Qd.device))[None, :]).sum(1)
    report("20 random hyperplane bits", torch.argsort(sig, stable=True))
