"""The reference-side binding (bindings/_b200.py -- what a maintainer would
add as pkg/src/mrpt/_kernels/_b200.py) keeps the reference kernels' calling
conventions and matches the oracle's kernels bit for bit."""

import importlib.util
import os

import numpy as np
import pytest

from conftest import ROOT, gaussian
from oracle import oracle as O
from paper_1509_06957_b200 import _native

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def b200():
    os.environ["MRPT_CUDA_LIB"] = _native.LIB_PATH
    spec = importlib.util.spec_from_file_location("_b200", os.path.join(ROOT, "bindings", "_b200.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_binding_kernels_match_oracle(b200, rng):
    X = gaussian(rng, 3000, 40)
    cp, rows, vals = O.sample_sparse_matrix(40, 6, 0.3, (5, 2))
    P = b200.project(X, cp, rows, vals)
    assert P.tobytes() == O.project(X, cp, rows, vals).tobytes()
    idx = O.grow_trees(X, 5, 6, 0.3, seed=5)
    Pq = np.stack([O.project(X[17:18], *R)[0] for R in idx["matrices"]])
    leaves = b200.route(Pq, idx["splits"])
    assert np.array_equal(leaves, O.route(Pq, idx["splits"]))
    n = X.shape[0]
    counts = np.zeros(n, np.int32)
    stamps = np.zeros(n, np.int64)
    out = np.empty(n, np.int64)
    m = b200.vote(idx["leaf_indices"], idx["leaf_offsets"], leaves, 2, counts, stamps, 3, out)
    assert np.array_equal(out[:m], O.candidates(leaves, idx, 2))
    assert np.array_equal(np.where(stamps == 3, counts, 0), O.vote_counts(leaves, idx))
    cand = np.arange(0, n, 7, dtype=np.int64)
    assert b200.scan(X, cand, X[5]).tobytes() == O.scan(X, cand, X[5]).tobytes()
    assert b200.fnv1a64(X.tobytes()) == O.fnv1a64(X.tobytes())
    assert b200.fnv1a64(b"foobar") == 0x85944171F73967E8
