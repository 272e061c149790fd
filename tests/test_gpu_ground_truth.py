"""f3: ground truth on the GPU (evaluation.py:28-100) against the reference's
own outputs (tests/golden/ground_truth.npz, written by the unmodified
reference) and the oracle, bit for bit: ids and float64 distances."""

import numpy as np
import pytest

import paper_1509_06957_b200 as mrpt
from conftest import golden
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def test_ground_truth_matches_reference_goldens():
    g = golden("ground_truth.npz")
    for name in g["names"]:
        X, Q, k = g[f"{name}_X"], g[f"{name}_Q"], int(g[f"{name}_k"])
        gt = mrpt.compute_ground_truth(X, Q, k)
        assert gt.k == k and gt.n_queries == Q.shape[0]
        assert np.array_equal(gt.indices, g[f"{name}_ids"]), name
        assert gt.distances.tobytes() == g[f"{name}_dists"].tobytes(), name
        assert gt.dataset_checksum == O.fnv1a64(X.tobytes())
        assert gt.query_checksum == O.fnv1a64(np.ascontiguousarray(Q, np.float32).tobytes())


def test_brute_force_k_above_n_and_float64_query():
    g = golden("ground_truth.npz")
    r = mrpt.brute_force_knn(g["kgtn_q"], 20, g["kgtn_X"])
    assert len(r) == 9 and r.shortfall == 11 and r.candidate_count == 9
    assert np.array_equal(r.indices, g["kgtn_ids"])
    assert r.distances.tobytes() == g["kgtn_dists"].tobytes()


def test_brute_force_errors_follow_reference():
    X = np.ones((5, 3), np.float32)
    with pytest.raises(mrpt.ParameterError):
        mrpt.brute_force_knn(np.zeros(3), 0, X)
    with pytest.raises(mrpt.ShapeError):
        mrpt.brute_force_knn(np.zeros(4), 2, X)
    with pytest.raises(mrpt.ShapeError):
        mrpt.compute_ground_truth(X, np.ones((2, 4), np.float32), 2)
    with pytest.raises(mrpt.ParameterError):
        mrpt.compute_ground_truth(X, np.ones((2, 3), np.float32), 6)


@pytest.mark.parametrize("n,d,nq,k", [(200_000, 128, 40, 100), (30_000, 784, 24, 10),
                                      (5_000, 33, 300, 1500), (1, 7, 3, 1)])
def test_ground_truth_matches_oracle_at_size(n, d, nq, k):
    """Multi-chunk merge, several passes (k > 512) and a one-row dataset."""
    rng = np.random.default_rng(n + d)
    c = 3.0 * rng.standard_normal((16, d))
    allx = (c[rng.integers(0, 16, size=n + nq)] + rng.standard_normal((n + nq, d))).astype(np.float32)
    X, Q = allx[:n], allx[n:]
    if n > 1:
        X[1::97] = X[0::97][:len(X[1::97])]  # exact duplicate rows: distance ties
    gt = mrpt.compute_ground_truth(X, Q, k)
    sel = range(0, nq, max(1, nq // 6))
    for i in sel:
        ids, dists, _ = O.brute_force_knn(X, Q[i], k)
        assert np.array_equal(gt.indices[i], ids)
        assert gt.distances[i].tobytes() == dists.tobytes()


def test_recall_helpers():
    truth = np.array([[1, 2, 3], [4, 5, 6]])
    got = np.array([[3, 2, 9], [-1, -1, -1]])
    assert mrpt.recall(got[0], truth[0]) == pytest.approx(2 / 3)
    assert mrpt.recall_batch(got, truth) == pytest.approx(1 / 3)
    with pytest.raises(mrpt.ParameterError):
        mrpt.recall(got[0], np.array([1, 1, 2]))


def test_candidate_set_equals_compiled_reference_order_as_a_set():
    """The compiled reference emits candidates in threshold-crossing order
    (_cy.pyx:57-78); this package returns the same set ascending (the numpy
    backend's order, _py.py:63-83)."""
    g = golden("candidates_unsorted.npz")
    index = mrpt.grow_trees(g["X"], int(g["n_trees"]), int(g["depth"]), seed=int(g["seed"]))
    b = g["bounds"]
    i = 0
    for v in g["votes"]:
        for q in g["Q"]:
            got, acc = mrpt.candidate_set(q, index, int(v))
            ref = g["cand"][b[i]:b[i + 1]]
            assert np.array_equal(got, np.sort(ref))
            assert np.all(np.diff(got) > 0)
            assert acc.counts()[ref].min() >= v if len(ref) else True
            i += 1
    acc.begin()  # a new epoch reads as all zeros until the next accumulate
    assert acc.counts().sum() == 0 and acc.count(int(ref[0]) if len(ref) else 0) == 0
