"""Build-time A/B in one process (TB=n in a spec fixes the trees per batch): grow_trees on a configuration twice per
variant (the first warms), variants chosen by environment settings given as
NAME=VAL[,NAME=VAL] arguments; also checks the variants build identical trees.
usage: python tools/build_ab.py CONFIG SCALE "MRPT_PROJ_D64=0" "MRPT_PROJ_D64=1" ...
(CACHED=1 in a spec: build from a Dataset whose checksum is already known,
i.e. the build without the K6 checksum.)"""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1509_06957_b200 as mrpt  # noqa: E402
from paper_1509_06957_b200 import workloads  # noqa: E402

cfg, scale = int(sys.argv[1]), float(sys.argv[2])
X, Q, p = workloads.generate(cfg, scale)
Xd = torch.from_numpy(X).cuda()
ref = None
for spec in sys.argv[3:]:
    for kv in spec.split(","):
        k, v = kv.split("=")
        os.environ[k] = v
    ts = []
    src = Xd
    if os.environ.get("CACHED") == "1":
        from paper_1509_06957_b200.core import as_dataset
        src = as_dataset(Xd)
        src.checksum
    tb = int(os.environ.get("TB", "0")) or None  # trees per K1+K5 batch (else: from free memory)
    for _ in range(2):
        index = D = None  # the previous index is freed first: the batch size depends on free memory
        gc.collect()
        torch.cuda.empty_cache()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        index = mrpt.grow_trees(src, p["n_trees"], p["depth"], p["sparsity"], seed=0, batch_trees=tb)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    D = index.device_index()
    sig = (D.splits.cpu().numpy().tobytes(), D.offsets.cpu().numpy().tobytes(),
           D.indices[:: max(1, p["n_trees"] // 7)].cpu().numpy().tobytes())
    same = ref is None or sig == ref
    ref = ref or sig
    print(f"config {cfg} scale {scale} [{spec}]: build {ts[-1]:.3f} s (first {ts[0]:.3f}) same={same}",
          flush=True)
    del index, D
