"""One grow_trees call on a generated workload (for ncu captures of the
build kernels K1/K5 and the checksum K6).  The first build warms the module;
MRPT_PROFILE_SECOND=1 builds twice so `--launch-skip` can target the second.
usage: python tools/profile_build.py [config] [scale]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1509_06957_b200 as mrpt  # noqa: E402
from paper_1509_06957_b200 import workloads  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
X, Q, p = workloads.generate(cfg, scale)
Xd = torch.from_numpy(X).cuda()
torch.cuda.synchronize()
t0 = time.perf_counter()
index = mrpt.grow_trees(Xd, p["n_trees"], p["depth"], p["sparsity"], seed=0)
torch.cuda.synchronize()
print(f"config {cfg} scale {scale}: n={X.shape[0]} d={X.shape[1]} T={p['n_trees']} l={p['depth']} "
      f"build {time.perf_counter() - t0:.3f} s", flush=True)
