"""The fused tcgen05 filter route (u8tc_bits: TMA-fed tcgen05.mma.kind::i8
into TMEM, bounds applied straight out of TMEM) returns exactly the oracle's
candidate counts, neighbour ids and float64 distances: several row tiles and
query blocks with ragged ends, K blocks ragged against the 128-byte TMA box,
u8 and s8 query quantisation, exact-tie masses (entry-list overflow -> exact
fallback), k at its limit, sparse and dense candidate bitmaps."""

import numpy as np
import pytest

import paper_1509_06957_b200 as mrpt
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _oracle(index, X, Q, k, v):
    ref = dict(matrices=[(R.col_ptr, R.row_idx, R.values) for R in index.matrices],
               splits=index.splits, leaf_offsets=index.leaf_offsets,
               leaf_indices=index.leaf_indices, depth=index.depth)
    return O.approximate_knn_batch(X, Q, k, ref, v)


def _data(kind, rng, n, d):
    if kind == "pixels":
        x = np.where(rng.random((n, d)) < 0.2, rng.random((n, d)), 0.0)
    elif kind == "ints":
        x = np.minimum(255, np.floor(rng.exponential(20.0, size=(n, d))))
    elif kind == "clusters01":
        c = rng.uniform(0, 0.5, size=(20, d))
        x = np.clip(c[rng.integers(0, 20, n)] + 0.05 * rng.standard_normal((n, d)), 0, 1)
    else:  # heavy duplicates
        base = rng.integers(0, 3, size=(40, d)).astype(np.float64)
        x = base[rng.integers(0, 40, n)]
    return x.astype(np.float32)


CASES = [
    # kind, n, d, nq, T, depth, k, v, shift
    ("pixels", 5000, 784, 300, 8, 5, 10, 1, 0.0),     # config-2 width: 7 K blocks (last ragged)
    ("pixels", 5000, 200, 260, 8, 5, 10, 1, -0.05),   # s8 queries, 2 K blocks
    ("ints", 4100, 128, 390, 10, 6, 10, 2, 0.0),      # exact u8 rows, one K block
    ("clusters01", 3000, 256, 385, 6, 4, 16, 1, 0.0), # k at the limit, ragged query block
    ("pixels", 2500, 1000, 300, 6, 4, 10, 1, 0.0),    # widest rows: 8 K blocks (ldq 1008)
    ("dups", 2000, 128, 300, 6, 5, 16, 1, 0.0),       # exact-tie masses: fallback path
    ("ints", 700, 160, 300, 5, 3, 1, 3, 0.0),         # k = 1, v > 1, n < 3 tiles
    ("pixels", 200, 256, 300, 3, 2, 10, 1, 0.0),      # n < one row tile
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-n{c[1]}-d{c[2]}-k{c[6]}-v{c[7]}")
def test_tc_route_parity(monkeypatch, rng, case):
    kind, n, d, nq, T, depth, k, v, shift = case
    monkeypatch.setenv("MRPT_SCAN_ROWS", "u8tc_bits")
    X = _data(kind, rng, n + nq, d)
    Xd, Q = X[:n], X[n:] + np.float32(shift)
    index = mrpt.grow_trees(Xd, T, depth, seed=5)
    ids, dists, counts = mrpt.approximate_knn_batch(Q, k, index, v)
    assert index.device_index().scan_choice.get((k, v)) == "u8tc_bits"
    rids, rd, rc = _oracle(index, Xd, Q, k, v)
    assert np.array_equal(counts.astype(np.int64), rc)
    assert np.array_equal(ids, rids)
    assert dists.tobytes() == rd.tobytes()


def test_tc_route_not_offered_outside_limits(rng):
    from paper_1509_06957_b200.search import _scan_variants

    X = _data("ints", rng, 3000, 64)          # ldq 64 < one 128-byte K block
    D = mrpt.grow_trees(X, 4, 4, seed=1).device_index()
    assert "u8tc_bits" not in _scan_variants(D, 10)
    X = _data("ints", rng, 3000, 128)
    D = mrpt.grow_trees(X, 4, 4, seed=1).device_index()
    assert "u8tc_bits" in _scan_variants(D, 16)
    assert "u8tc_bits" not in _scan_variants(D, 17)   # k smallest bounds in shared memory: k <= 16


@pytest.mark.parametrize("route", ["u8tc_bits", "u8"])
def test_host_batch_pipelined_paths(rng, route):
    """Host batches >= 4096 queries take the overlapped paths: bitmap routes
    upload in pieces, route + vote each piece as it lands and run one
    filter over the whole batch; list routes pipeline whole pieces.  Same
    answers as the oracle either way."""
    n, d, nq, k, v = 3000, 136, 4500, 10, 1
    X = _data("ints", rng, n + nq, d)
    Xd, Q = X[:n], X[n:]
    index = mrpt.grow_trees(Xd, 6, 5, seed=13)
    index.device_index().pin_route(k, v, route)
    ids, dists, counts = mrpt.approximate_knn_batch(Q, k, index, v)
    rids, rd, rc = _oracle(index, Xd, Q, k, v)
    assert np.array_equal(counts.astype(np.int64), rc)
    assert np.array_equal(ids, rids)
    assert dists.tobytes() == rd.tobytes()


def test_tc_dot_products_equal_reference_dots(tmp_path):
    """Debug mode of the fused kernel (MRPT_TC_DEBUG): every (query, row)
    int32 dot product it reads out of TMEM is compared on the device with a
    naive int32 loop over the same s8 operands -- they must agree exactly
    (the admission rule's bounds rest on that)."""
    import os
    import subprocess
    import sys
    import textwrap

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = textwrap.dedent("""
        import numpy as np, sys
        sys.path.insert(0, %r)
        import paper_1509_06957_b200 as mrpt
        rng = np.random.default_rng(3)
        X = np.where(rng.random((3500, 300)) < 0.3, rng.random((3500, 300)), 0).astype(np.float32)
        Q = X[3000:] - np.float32(0.02)   # signed queries too
        index = mrpt.grow_trees(X[:3000], 5, 4, seed=1)
        index.device_index().pin_route(10, 1, "u8tc_bits")
        mrpt.approximate_knn_batch(Q, 10, index, 1)
        index2 = mrpt.grow_trees(X[:3000], 5, 4, seed=2)
        index2.device_index().pin_route(10, 1, "u8tc_bits")
        mrpt.approximate_knn_batch(np.abs(X[3000:]), 10, index2, 1)
    """ % root)
    env = dict(os.environ, MRPT_TC_DEBUG="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stderr.splitlines() if "D mismatches=" in l]
    assert len(lines) >= 2
    assert all("D mismatches=0 " in l for l in lines), lines


def test_tc_route_several_query_chunks(rng):
    """More queries than one fused-filter chunk (16384): the per-chunk
    bookkeeping (entry lists, shared bounds, bound lists) is reset and
    offset per chunk; answers equal the oracle's."""
    import torch

    from paper_1509_06957_b200.search import query_device

    n, d, nq, k, v = 1500, 128, 20000, 5, 1
    X = _data("ints", rng, n + nq, d)
    Xd, Q = X[:n], X[n:]
    index = mrpt.grow_trees(Xd, 4, 4, seed=17)
    D = index.device_index()
    D.pin_route(k, v, "u8tc_bits")
    ids, dists, counts = (t.cpu().numpy() for t in query_device(D, torch.from_numpy(Q).cuda(), k, v))
    rids, rd, rc = _oracle(index, Xd, Q, k, v)
    assert np.array_equal(counts.astype(np.int64), rc)
    assert np.array_equal(ids, rids)
    assert dists.tobytes() == rd.tobytes()
