"""Seeded fuzz over shapes, thresholds, k and every exact filter route: each
case must return exactly the oracle's candidate counts, ids and float64
distances (the reference's algorithm, oracle/oracle.py).  Deterministic: the
cases are drawn from a fixed seed."""

import numpy as np
import pytest

import paper_1509_06957_b200 as mrpt
from oracle import oracle as O

pytestmark = pytest.mark.gpu

ROUTES = ["auto", "u8", "u8tc_bits", "fp16", "fp32"]


def _cases():
    rng = np.random.default_rng(1509)
    out = []
    for i in range(24):
        n = int(rng.integers(50, 6000))
        d = int(rng.choice([3, 8, 17, 32, 64, 100, 128, 260]))
        T = int(rng.integers(1, 40))
        depth = int(rng.integers(1, max(2, min(9, int(np.log2(n))) + 1)))
        v = int(rng.integers(1, T + 1))
        k = int(rng.choice([1, 3, 10, 33, 96, 150]))
        kind = str(rng.choice(["gauss", "ints", "nonneg", "dups"]))
        route = ROUTES[i % len(ROUTES)]
        out.append((i, n, d, T, depth, v, k, kind, route))
    return out


def _data(kind, rng, n, d):
    if kind == "gauss":
        return rng.standard_normal((n, d)).astype(np.float32)
    if kind == "ints":
        return rng.integers(0, 256, size=(n, d)).astype(np.float32)
    if kind == "nonneg":
        return np.abs(rng.standard_normal((n, d))).astype(np.float32)
    base = rng.integers(0, 3, size=(max(2, n // 50), d)).astype(np.float32)
    return base[rng.integers(0, base.shape[0], n)]


def _offered(index, k):
    from paper_1509_06957_b200.search import _scan_variants

    return _scan_variants(index.device_index(), k)


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"c{c[0]}-{c[8]}")
def test_fuzz_matches_oracle(monkeypatch, case):
    i, n, d, T, depth, v, k, kind, route = case
    if route != "auto":
        monkeypatch.setenv("MRPT_SCAN_ROWS", route)
    if route == "fp16":
        monkeypatch.setenv("MRPT_FP16_FILTER", "1")
    rng = np.random.default_rng(1000 + i)
    nq = int(rng.integers(256, 600))  # >= 256: the route autotune (and its forcing) runs
    X = _data(kind, rng, n + nq, d)
    Xd, Q = X[:n], X[n:]
    index = mrpt.grow_trees(Xd, T, depth, seed=i)
    ids, dists, counts = mrpt.approximate_knn_batch(Q, k, index, v)
    chosen = index.device_index().scan_choice.get((k, v))
    if route not in ("auto",) and route in _offered(index, k):
        assert chosen == route
    ref = dict(matrices=[(R.col_ptr, R.row_idx, R.values) for R in index.matrices],
               splits=index.splits, leaf_offsets=index.leaf_offsets,
               leaf_indices=index.leaf_indices, depth=depth)
    rids, rd, rc = O.approximate_knn_batch(Xd, Q, k, ref, v)
    assert np.array_equal(counts.astype(np.int64), rc)
    assert np.array_equal(ids, rids)
    assert dists.tobytes() == rd.tobytes()


def _tc_cases():
    rng = np.random.default_rng(2048)
    out = []
    for i in range(12):
        n = int(rng.integers(100, 9000))
        d = int(rng.choice([128, 132, 200, 256, 384, 520, 784, 1000, 1024]))
        T = int(rng.integers(1, 24))
        depth = int(rng.integers(1, max(2, min(8, int(np.log2(n))) + 1)))
        v = int(rng.integers(1, min(T, 3) + 1))
        k = int(rng.integers(1, 17))
        kind = str(rng.choice(["ints", "nonneg", "dups", "shifted"]))
        out.append((i, n, d, T, depth, v, k, kind))
    return out


@pytest.mark.parametrize("case", _tc_cases(), ids=lambda c: f"tc{c[0]}-n{c[1]}-d{c[2]}-k{c[6]}")
def test_fuzz_tc_route(case):
    """Seeded fuzz of the fused tcgen05 filter route (pinned): ragged row
    tiles and query blocks (odd cluster pairs), every K-block count, k up to
    its limit, signed (shifted) queries, duplicate masses."""
    i, n, d, T, depth, v, k, kind = case
    rng = np.random.default_rng(5000 + i)
    nq = int(rng.integers(256, 900))
    X = _data("nonneg" if kind == "shifted" else kind, rng, n + nq, d)
    Xd, Q = X[:n], X[n:]
    if kind == "shifted":
        Q = Q - np.float32(0.1)
    index = mrpt.grow_trees(Xd, T, depth, seed=i)
    index.device_index().pin_route(k, v, "u8tc_bits")
    ids, dists, counts = mrpt.approximate_knn_batch(Q, k, index, v)
    ref = dict(matrices=[(R.col_ptr, R.row_idx, R.values) for R in index.matrices],
               splits=index.splits, leaf_offsets=index.leaf_offsets,
               leaf_indices=index.leaf_indices, depth=depth)
    rids, rd, rc = O.approximate_knn_batch(Xd, Q, k, ref, v)
    assert np.array_equal(counts.astype(np.int64), rc)
    assert np.array_equal(ids, rids)
    assert dists.tobytes() == rd.tobytes()
