"""Probe: the fused tcgen05 filter (u8tc_bits) against the library-GEMM
bitmap route (u8gemm_bits) on a BASELINE config: identical answers, and the
event-timed K4 stage of each (not a bench number)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1509_06957_b200 as mrpt  # noqa: E402
from paper_1509_06957_b200 import search, workloads  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    v = int(sys.argv[3]) if len(sys.argv) > 3 else None
    X, Q, p = workloads.generate(cfg, scale=scale)
    index = mrpt.grow_trees(X, p["n_trees"], p["depth"], sparsity=p["sparsity"], seed=0)
    D = index.device_index()
    Qd = torch.from_numpy(Q).cuda()
    k = p["k"]
    v = v if v is not None else p["headline_votes"]
    res = {}
    runs = [("u8gemm_bits", None)] + [("u8tc_bits", cg) for cg in (1, 2, 4)]
    for route, cg in runs:
        if cg is not None:
            os.environ["MRPT_TC_CG"] = str(cg)
            os.environ["MRPT_TC_DEBUG"] = "1"
            search.query_device(D, Qd, k, v)
            torch.cuda.synchronize()
            del os.environ["MRPT_TC_DEBUG"]
        D.pin_route(k, v, route)
        out = search.query_device(D, Qd, k, v)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            out = search.query_device(D, Qd, k, v)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[(route, cg)] = [t.cpu() for t in out]
        print(f"{route} cg={cg}: {min(ts):.3f} ms per {Qd.shape[0]} queries (min of 5)", flush=True)
    a = res[("u8gemm_bits", None)]
    for key, b in res.items():
        print(key, "ids equal:", bool(torch.equal(a[0], b[0])), "dists equal:",
              bool(torch.equal(a[1], b[1])), "counts equal:", bool(torch.equal(a[2], b[2])))


if __name__ == "__main__":
    main()
