"""Shared fixtures.  `-m gpu` tests need a CUDA device and the built library;
everything else runs on the CPU (the oracle, host logic, the ABI surface)."""

import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libmrpt_cuda.so")
    config.addinivalue_line("markers", "slow: larger parity cases")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        have_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this environment")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def golden(name):
    with np.load(os.path.join(GOLDEN, name), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def golden_small_names():
    return sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "small_*.npz")))


def unpack_matrices(g):
    """Per-tree (col_ptr, rows, vals) of a golden record."""
    out, off = [], 0
    for t, nnz in enumerate(g["mat_nnz"]):
        nnz = int(nnz)
        out.append((g["mat_col_ptr"][t], g["mat_rows"][off:off + nnz], g["mat_vals"][off:off + nnz]))
        off += nnz
    return out


def gaussian(rng, n, d):
    return rng.standard_normal((n, d)).astype(np.float32)


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)
