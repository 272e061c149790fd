"""Every exact K4 filter variant (u8 shadow with dp4a, fp16 shadow, float32)
returns exactly the oracle's neighbours and distances: non-negative float
data, integer-valued data (exact u8 shadow), queries with negative values
(s8 query quantisation), signed data (no u8 shadow: the float32 filter),
heavy exact ties (buffer overflow -> exact tiled fallback), k up to 120 and
the >120 multi-pass path."""

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
        x = np.where(rng.random((n, d)) < 0.3, rng.random((n, d)), 0.0)
    elif kind == "ints":
        x = np.minimum(255, np.floor(rng.exponential(20.0, size=(n, d))))
    elif kind == "clusters01":
        c = rng.uniform(0, 0.5, size=(20, d))
        x = np.clip(c[rng.integers(0, 20, n)] + 0.05 * rng.standard_normal((n, d)), 0, 1)
    elif kind == "signed":
        x = rng.standard_normal((n, d))
    else:  # heavy duplicates
        base = rng.integers(0, 3, size=(40, d)).astype(np.float64)
        x = base[rng.integers(0, 40, n)]
    return x.astype(np.float32)


@pytest.mark.parametrize("variant", ["u8", "u8tc_bits", "fp16", "fp32"])
@pytest.mark.parametrize("kind,d,k,v", [("pixels", 96, 10, 1), ("ints", 128, 10, 2),
                                         ("clusters01", 256, 10, 2), ("signed", 64, 7, 1),
                                         ("dups", 32, 20, 1), ("pixels", 200, 100, 1)])
def test_variant_parity(monkeypatch, rng, variant, kind, d, k, v):
    if variant == "u8tc_bits" and (k > 16 or d < 128):
        pytest.skip("the fused tcgen05 filter takes k <= 16 and rows of >= 128 bytes")
    monkeypatch.setenv("MRPT_SCAN_ROWS", variant)
    if variant == "fp16":
        monkeypatch.setenv("MRPT_FP16_FILTER", "1")
    n, nq = 4000, 300
    X = _data(kind, rng, n + nq, d)
    Xd, Q = X[:n], X[n:]
    if kind == "pixels":
        Q = Q - 0.05  # negative query coordinates: s8 query quantisation
    index = mrpt.grow_trees(Xd, 6, 6, seed=3)
    ids, dists, counts = mrpt.approximate_knn_batch(Q, k, index, v)
    allowed = (variant, "fp32")
    assert index.device_index().scan_choice.get((k, v)) in allowed
    rids, rd, rc = _oracle(index, Xd, Q, k, v)
    assert np.array_equal(counts.astype(np.int64), rc)
    assert np.array_equal(ids, rids)
    assert dists.tobytes() == rd.tobytes()


def test_large_k_batch_multipass(rng):
    X = _data("pixels", rng, 3000, 64)
    index = mrpt.grow_trees(X[:2700], 4, 2, seed=1)
    ids, dists, counts = mrpt.approximate_knn_batch(X[2700:2710], 500, index, 1)
    rids, rd, rc = _oracle(index, X[:2700], X[2700:2710], 500, 1)
    assert np.array_equal(ids, rids) and dists.tobytes() == rd.tobytes()


@pytest.mark.parametrize("v,k", [(6, 8), (5, 16), (1, 16)])
def test_bitmap_route_edges(monkeypatch, rng, v, k):
    """The bitmap hand-over + fused tcgen05 filter at the edges: v = T (mostly
    empty candidate sets), k larger than most candidate sets (-1 / inf
    padding), k at its limit; a foreign index with unsorted leaf slices; n
    not a multiple of 32."""
    monkeypatch.setenv("MRPT_SCAN_ROWS", "u8tc_bits")
    n, d, nq = 3001, 140, 300
    X = _data("ints", rng, n + nq, d)
    Xd, Q = X[:n], X[n:]
    a = mrpt.grow_trees(Xd, 6, 6, seed=21)
    li = a.leaf_indices.copy()
    for t in range(6):
        o = a.leaf_offsets[t]
        for j in range(len(o) - 1):
            li[t, o[j]:o[j + 1]] = li[t, o[j]:o[j + 1]][rng.permutation(o[j + 1] - o[j])]
    b = mrpt.MRPTIndex(dataset=mrpt.Dataset(Xd), n_trees=6, depth=6, sparsity=a.sparsity, seed=21,
                       fixed_count=False, matrices=a.matrices, splits=a.splits,
                       leaf_offsets=a.leaf_offsets, leaf_indices=li,
                       dataset_checksum=a.dataset_checksum)
    for index in (a, b):
        ids, dists, counts = mrpt.approximate_knn_batch(Q, k, index, v)
        assert index.device_index().scan_choice.get((k, v)) == "u8tc_bits"
        rids, rd, rc = _oracle(index, Xd, Q, k, v)
        assert np.array_equal(counts.astype(np.int64), rc)
        assert np.array_equal(ids, rids)
        assert dists.tobytes() == rd.tobytes()


@pytest.mark.parametrize("variant", ["u8", "u8tc_bits"])
def test_u8_routes_odd_width(monkeypatch, rng, variant):
    """d not a multiple of 4: the u8 list route falls back to the float32
    filter inside the library, the bitmap route is not offered; answers stay
    exact."""
    monkeypatch.setenv("MRPT_SCAN_ROWS", variant)
    n, d, nq = 2500, 37, 280
    X = _data("ints", rng, n + nq, d)
    Xd, Q = X[:n], X[n:]
    index = mrpt.grow_trees(Xd, 5, 5, seed=2)
    ids, dists, counts = mrpt.approximate_knn_batch(Q, 9, index, 1)
    rids, rd, rc = _oracle(index, Xd, Q, 9, 1)
    assert np.array_equal(ids, rids)
    assert dists.tobytes() == rd.tobytes()


@pytest.mark.parametrize("d,k,v", [(64, 10, 1), (256, 25, 2), (37, 9, 1), (200, 100, 1)])
def test_signed_data_routes(rng, d, k, v):
    """Signed data has no u8 shadow: the autotune chooses among the float32
    (and, when wide, fp16) filters; exactly the oracle's answers, including
    odd widths and k near the filters' limit."""
    n, nq = 4000, 290
    X = _data("signed", rng, n + nq, d)
    Xd, Q = X[:n], X[n:]
    index = mrpt.grow_trees(Xd, 6, 5, seed=9)
    ids, dists, counts = mrpt.approximate_knn_batch(Q, k, index, v)
    assert index.device_index().scan_choice.get((k, v)) in ("fp16", "fp32")
    rids, rd, rc = _oracle(index, Xd, Q, k, v)
    assert np.array_equal(counts.astype(np.int64), rc)
    assert np.array_equal(ids, rids)
    assert dists.tobytes() == rd.tobytes()
