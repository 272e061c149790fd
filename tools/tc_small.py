"""Small fused-filter run (memcheck target): ragged tiles / query blocks."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1509_06957_b200 as mrpt  # noqa: E402

rng = np.random.default_rng(1)
X = np.where(rng.random((1700, 200)) < 0.3, rng.random((1700, 200)), 0).astype(np.float32)
index = mrpt.grow_trees(X[:1400], 4, 4, seed=3)
index.device_index().pin_route(10, 1, "u8tc_bits")
ids, d, c = mrpt.approximate_knn_batch(X[1400:], 10, index, 1)
print("ok", ids.shape, int(c.sum()))
