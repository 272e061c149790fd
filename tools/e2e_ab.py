"""Interleaved in-process A/B of the host-batch pipeline knobs (e2e through
approximate_knn_batch with pinned host queries).  The knobs are read from the
environment on every call, so the settings alternate round by round inside
one process and host jitter hits all of them alike.

usage: python tools/e2e_ab.py [config] [rounds] "ENV=1 ENV2=2" "ENV=2" ...
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1509_06957_b200 as mrpt  # noqa: E402
from paper_1509_06957_b200 import workloads  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    settings = [dict(kv.split("=", 1) for kv in s.split()) for s in sys.argv[3:]] or [{}]
    X, Q, p = workloads.generate(cfg)
    index = mrpt.grow_trees(X, p["n_trees"], p["depth"], p["sparsity"], seed=0)
    k, v = p["k"], p["headline_votes"]
    Qpin = torch.from_numpy(Q).pin_memory()
    ref = mrpt.approximate_knn_batch(Qpin, k, index, v)  # autotune + warm-up
    calls = 10
    times = [[] for _ in settings]
    for r in range(rounds):
        for i, s in enumerate(settings):
            saved = {key: os.environ.get(key) for key in s}
            os.environ.update(s)
            for _ in range(3):
                out = mrpt.approximate_knn_batch(Qpin, k, index, v)
            if r == 0:
                assert all(np.array_equal(a, b) for a, b in zip(out, ref)), s
            t0 = time.perf_counter()
            for _ in range(calls):
                mrpt.approximate_knn_batch(Qpin, k, index, v)
            times[i].append(time.perf_counter() - t0)
            for key, val in saved.items():
                if val is None:
                    os.environ.pop(key, None)
                else:
                    os.environ[key] = val
    for s, t in zip(settings, times):
        qps = [p["nq"] * calls / x for x in t]
        print(f"{s}: median {np.median(qps):,.0f} q/s  best {max(qps):,.0f}  worst {min(qps):,.0f}")


if __name__ == "__main__":
    main()
