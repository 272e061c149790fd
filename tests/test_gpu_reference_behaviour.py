"""The reference package's behavioural contract, exercised on the GPU path.

Each test restates a property the reference's own suite pins (file:line of
the reference test in the docstring) and checks it against this package.
"""

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import paper_1509_06957_b200 as mrpt
from conftest import gaussian
from oracle import oracle as O
from paper_1509_06957_b200.search import _route_tree

pytestmark = pytest.mark.gpu


def _matrix(dense):
    """SparseProjectionMatrix holding exactly the non-zeros of a dense d x depth array."""
    arr = np.asarray(dense, dtype=np.float32)
    d, depth = arr.shape
    cols = [np.flatnonzero(arr[:, j]) for j in range(depth)]
    ptr = np.concatenate([[0], np.cumsum([len(c) for c in cols])]).astype(np.int64)
    rows = np.concatenate(cols).astype(np.int32) if ptr[-1] else np.zeros(0, np.int32)
    vals = (np.concatenate([arr[c, j] for j, c in enumerate(cols)]).astype(np.float32)
            if ptr[-1] else np.zeros(0, np.float32))
    return mrpt.SparseProjectionMatrix(d=d, depth=depth, a=1.0, seed=0, col_ptr=ptr, row_idx=rows,
                                       values=vals)


def _tree(depth, splits, offsets, ids, matrix):
    return mrpt.RPTree(random_matrix=matrix, depth=depth,
                       splits=np.asarray(splits, np.float32),
                       leaf_offsets=np.asarray(offsets, np.int64),
                       leaf_indices=np.asarray(ids, np.int32))


def _index(X, trees):
    X = mrpt.Dataset(X)
    return mrpt.MRPTIndex(dataset=X, n_trees=len(trees), depth=trees[0][0].depth, sparsity=1.0,
                          seed=0, fixed_count=False, matrices=[t[0] for t in trees],
                          splits=np.stack([np.asarray(t[1], np.float32) for t in trees]),
                          leaf_offsets=np.stack([np.asarray(t[2], np.int64) for t in trees]),
                          leaf_indices=np.stack([np.asarray(t[3], np.int32) for t in trees]),
                          dataset_checksum=X.checksum)


# --- median_split / build_tree (reference tests/test_trees.py:26-111) ---------
def test_median_split_cases():
    s, left, right = mrpt.median_split(np.array([3.0, 1.0, 2.0, 4.0]), np.array([0, 1, 2, 3]))
    assert s == 2.0 and set(left) == {1, 2} and set(right) == {0, 3}
    s, left, right = mrpt.median_split(np.array([5.0, 4.0, 3.0, 2.0, 1.0]), np.arange(5))
    assert s == 3.0 and len(left) == 3 and len(right) == 2
    s, left, right = mrpt.median_split(np.array([7.0, 7.0]), np.array([0, 1]))
    assert s == 7.0 and set(left) == {0, 1} and len(right) == 0


def test_median_split_against_sorting(rng):
    for _ in range(30):
        m = int(rng.integers(2, 60))
        v = rng.standard_normal(m).astype(np.float32)
        s, left, right = mrpt.median_split(v, np.arange(m))
        assert s == np.sort(v)[(m + 1) // 2 - 1]
        assert left.tolist() == np.flatnonzero(v <= s).tolist()  # stable order too
        assert right.tolist() == np.flatnonzero(v > s).tolist()


def test_build_tree_hand_cases(rng):
    splits, offsets, order = mrpt.build_tree(gaussian(rng, 6, 1), depth=0, indices=[3, 1, 4])
    assert splits.size == 0 and list(offsets) == [0, 3] and list(order) == [3, 1, 4]
    splits, offsets, order = mrpt.build_tree(np.array([[1.0], [2.0], [3.0], [4.0]]), depth=1)
    assert splits.tolist() == [2.0]
    assert set(order[offsets[0]:offsets[1]]) == {0, 1}
    splits, offsets, order = mrpt.build_tree(np.full((4, 1), 7.0, np.float32), depth=1)
    assert splits.tolist() == [7.0] and offsets.tolist() == [0, 4, 4]
    P = np.array([[5.0, 1.0], [5.0, 2.0], [5.0, 3.0], [5.0, 4.0]], dtype=np.float32)
    splits, offsets, order = mrpt.build_tree(P, depth=2)
    sizes = np.diff(offsets)
    assert sizes.sum() == 4 and sizes[2] == 0 and sizes[3] == 0


def test_build_tree_matches_oracle_with_custom_indices(rng):
    P = gaussian(rng, 50, 4)
    idx = rng.permutation(50)[:37]
    s, o, order = mrpt.build_tree(P, 4, indices=idx)
    rs, ro, rpos = O.build_tree(P[idx], 4)
    assert s.tobytes() == rs.tobytes() and np.array_equal(o, ro)
    assert np.array_equal(order, idx[rpos])


# --- grow_trees (test_trees.py:117-216) -----------------------------------------
def test_full_depth_singletons_and_validation(rng):
    X = gaussian(rng, 8, 5)
    index = mrpt.grow_trees(X, n_trees=2, depth=3, sparsity=1.0, seed=11)
    for t in range(2):
        tree = index.tree(t)
        leaves = [tree.leaf(i) for i in range(tree.n_leaves)]
        assert all(len(x) == 1 for x in leaves)
        assert sorted(np.concatenate(leaves).tolist()) == list(range(8))


def test_determinism_and_distinct_matrices(rng):
    X = gaussian(rng, 64, 10)
    a = mrpt.grow_trees(X, 4, 4, seed=123)
    b = mrpt.grow_trees(X, 4, 4, seed=123)
    assert a.splits.tobytes() == b.splits.tobytes()
    assert np.array_equal(a.leaf_indices, b.leaf_indices)
    c = mrpt.grow_trees(gaussian(rng, 32, 8), 3, 2, sparsity=1.0, seed=4)
    assert len({c.matrices[t].values.tobytes() for t in range(3)}) == 3


def test_threads_argument_and_env(rng, monkeypatch):
    X = gaussian(rng, 128, 12)
    serial = mrpt.grow_trees(X, 6, 4, seed=5, threads=1)
    threaded = mrpt.grow_trees(X, 6, 4, seed=5, threads=4)
    assert np.array_equal(serial.leaf_indices, threaded.leaf_indices)
    monkeypatch.setenv("MRPT_THREADS", "3")
    env = mrpt.grow_trees(X, 6, 4, seed=5)
    assert np.array_equal(env.splits, serial.splits)


def test_partition_and_balance(rng):
    for _ in range(15):
        n = int(rng.integers(16, 700))
        depth = int(rng.integers(1, min(6, int(math.log2(n))) + 1))
        X = gaussian(rng, n, int(rng.integers(2, 24)))
        index = mrpt.grow_trees(X, 2, depth, sparsity=1.0, seed=int(rng.integers(1 << 30)))
        lo, hi = n // 2 ** depth, -(-n // 2 ** depth)
        for t in range(2):
            tree = index.tree(t)
            assert np.array_equal(np.sort(tree.leaf_indices), np.arange(n))
            assert set(np.unique(tree.leaf_sizes())).issubset({lo, hi})


def test_duplicate_points_pile_into_leftmost_leaf():
    X = np.ones((16, 4), dtype=np.float32)
    index = mrpt.grow_trees(mrpt.Dataset(X), 2, 3, seed=1)
    for t in range(2):
        assert index.tree(t).leaf_sizes()[0] == 16


def test_memory_and_bounds(rng):
    index = mrpt.grow_trees(gaussian(rng, 64, 10), 4, 4, seed=2)
    assert index.memory_bytes() >= index.splits.nbytes + index.leaf_indices.nbytes
    assert index.max_candidates() == 4 * math.ceil(64 / 16)


# --- routing (test_search.py:76-111) ---------------------------------------------
def test_points_route_to_their_own_leaf(rng):
    for seed in (1, 2):
        n = int(rng.integers(20, 300))
        X = gaussian(rng, n, 15)
        index = mrpt.grow_trees(X, 5, int(rng.integers(1, 5)), seed=seed)
        # batched: each point's leaf in every tree contains the point
        from paper_1509_06957_b200 import _device
        from paper_1509_06957_b200.search import _route_device

        leaves = _device.d2h(_route_device(_device.h2d(X), index.device_index()))
        for t in range(index.n_trees):
            o, li = index.leaf_offsets[t], index.leaf_indices[t]
            for i in range(n):
                assert i in li[o[leaves[i, t]]:o[leaves[i, t] + 1]]
        assert 0 in mrpt.tree_query(X[0], index.tree(0))


def test_hand_built_routing():
    m = _matrix(np.eye(4, 2))
    tree = _tree(2, [0.0, -1.0, 5.0], [0, 1, 2, 3, 4], [0, 1, 2, 3], m)
    assert mrpt.tree_query(np.array([-10.0, -10.0, 0.0, 0.0], np.float32), tree).tolist() == [0]
    m1 = _matrix(np.array([[1.0], [0.0], [0.0]]))
    tree = _tree(1, [0.0], [0, 2, 4], [0, 1, 2, 3], m1)
    assert set(mrpt.tree_query(np.array([-1.0, 9.0, 9.0], np.float32), tree)) == {0, 1}
    assert set(mrpt.tree_query(np.array([0.5, 0.0, 0.0], np.float32), tree)) == {2, 3}
    tree = _tree(1, [2.0], [0, 1, 2], [0, 1], _matrix(np.array([[1.0]])))
    assert mrpt.tree_query(np.array([2.0], np.float32), tree).tolist() == [0]  # <= goes left


# --- voting and the exact stage (test_search.py:117-305) ------------------------
def _three_tree_fixture():
    X = np.array([[0.0, 0.0], [1.0, 0.0], [2.0, 0.0], [10.0, 0.0]], dtype=np.float32)
    m = _matrix(np.zeros((2, 1)))
    trees = []
    for left in [(1, 2), (1, 3), (1, 2)]:
        right = tuple(i for i in range(4) if i not in left)
        trees.append((m, [0.0], [0, 2, 4], list(left) + list(right)))
    return X, _index(X, trees)


def test_vote_threshold_fixture():
    X, index = _three_tree_fixture()
    q = np.array([0.9, 0.0], dtype=np.float32)
    cands, _ = mrpt.candidate_set(q, index, votes=2)
    assert set(cands.tolist()) == {1, 2}
    r = mrpt.approximate_knn(q, 2, index, votes=2)
    assert r.indices.tolist() == [1, 2] and r.candidate_count == 2
    cands, _ = mrpt.candidate_set(q, index, votes=1)
    assert set(cands.tolist()) == {1, 2, 3}


def test_single_tree_single_vote_is_defeatist(rng):
    X = gaussian(rng, 100, 8)
    index = mrpt.grow_trees(X, 1, 3, seed=6)
    q = gaussian(rng, 1, 8)[0]
    leaf = mrpt.tree_query(q, index.tree(0))
    exp = mrpt.exact_knn_in_set(q, 5, leaf, index.dataset)
    got = mrpt.approximate_knn(q, 5, index, votes=1)
    assert got.indices.tolist() == exp.indices.tolist()
    assert got.distances.tolist() == exp.distances.tolist()


def test_argument_errors_in_reference_order(rng):
    index = mrpt.grow_trees(gaussian(rng, 32, 6), 4, 2, seed=1)
    q = gaussian(rng, 1, 6)[0]
    with pytest.raises(mrpt.ParameterError):
        mrpt.approximate_knn(q, 3, index, votes=0)
    with pytest.raises(mrpt.ParameterError):
        mrpt.approximate_knn(q, 3, index, votes=5)
    with pytest.raises(mrpt.ParameterError):
        mrpt.approximate_knn(q, 0, index, votes=1)
    with pytest.raises(mrpt.ShapeError):
        mrpt.approximate_knn(np.zeros(5, np.float32), 3, index, votes=1)
    with pytest.raises(mrpt.ShapeError):
        mrpt.approximate_knn_batch(np.zeros((2, 5), np.float32), 3, index, votes=1)


def test_shortfall_and_empty_results(rng):
    index = mrpt.grow_trees(gaussian(rng, 64, 6), 2, 4, seed=8)
    r = mrpt.approximate_knn(gaussian(rng, 1, 6)[0], 50, index, votes=2)
    assert len(r) == r.candidate_count <= 8 and r.shortfall == 50 - len(r)
    r = mrpt.exact_knn_in_set(gaussian(rng, 1, 3)[0], 4, np.empty(0, np.int64), gaussian(rng, 10, 3))
    assert len(r) == 0 and r.candidate_count == 0
    X = np.ones((16, 4), dtype=np.float32)
    dup = mrpt.grow_trees(mrpt.Dataset(X), 2, 3, seed=1)
    for scale in (3.0, -3.0, 0.0):
        q = np.full(4, scale, np.float32)
        for t in range(dup.n_trees):
            assert len(mrpt.tree_query(q, dup.tree(t))) in (0, 16)
        r = mrpt.approximate_knn(q, 4, dup, votes=1)
        assert len(r) <= 4 and r.candidate_count in (0, 16)


def test_exact_scan_contract(rng):
    X = gaussian(rng, 80, 7)
    q = gaussian(rng, 1, 7)[0]
    full = mrpt.exact_knn_in_set(q, 10, np.arange(80), X)
    d2 = ((X.astype(np.float64) - q.astype(np.float64)) ** 2).sum(axis=1)
    assert full.indices.tolist() == np.lexsort((np.arange(80), d2))[:10].tolist()
    Xt = np.array([[0.0, 1.0], [1.0, 0.0], [5.0, 5.0]], dtype=np.float32)
    assert mrpt.exact_knn_in_set(np.zeros(2), 1, np.array([1, 0]), Xt).indices.tolist() == [0]
    assert mrpt.exact_knn_in_set(np.zeros(2), 2, np.array([1, 0]), Xt).indices.tolist() == [0, 1]
    with pytest.raises(mrpt.IntegrityError):
        mrpt.exact_knn_in_set(q[:3], 2, np.array([0, 10]), gaussian(rng, 10, 3))
    with pytest.raises(mrpt.IntegrityError):
        mrpt.exact_knn_in_set(q[:3], 2, np.array([-1]), gaussian(rng, 10, 3))
    r = mrpt.exact_knn_in_set(q[:5], 100, np.arange(12), gaussian(rng, 12, 5))
    assert len(r) == 12 and (np.diff(r.distances) >= 0).all()


def test_independent_python_scan_oracle():
    """test_acceptance.py:57-78: plain-python sums, (distance, index) order."""
    rng = np.random.default_rng(101)
    for _ in range(10):
        n, d = int(rng.integers(1, 201)), int(rng.integers(1, 17))
        X = gaussian(rng, n, d)
        q = gaussian(rng, 1, d)[0]
        scored = sorted((sum((float(a) - float(b)) ** 2 for a, b in zip(row, q)), i)
                        for i, row in enumerate(X))
        for k in (1, 5, n):
            got = mrpt.exact_knn_in_set(q, k, np.arange(n), X)
            assert got.indices.tolist() == [i for _, i in scored[:min(k, n)]]


def test_candidate_bound_nesting_and_counts(rng):
    X = gaussian(rng, 300, 10)
    index = mrpt.grow_trees(X, 6, 3, seed=14)
    bound = index.max_candidates()
    for _ in range(6):
        q = gaussian(rng, 1, 10)[0]
        prev = None
        for v in range(1, index.n_trees + 1):
            cands, acc = mrpt.candidate_set(q, index, votes=v)
            assert len(cands) <= bound
            cur = set(cands.tolist())
            assert prev is None or cur <= prev
            prev = cur
        _, acc = mrpt.candidate_set(q, index, votes=1)
        counts = acc.counts()
        touched = sum(len(mrpt.tree_query(q, index.tree(t))) for t in range(index.n_trees))
        assert counts.sum() == touched and counts.max() <= index.n_trees
        x = int(rng.integers(0, 300))
        recount = sum(_route_tree(np.ascontiguousarray(X[x]), index.tree(t)) ==
                      _route_tree(q, index.tree(t)) for t in range(index.n_trees))
        assert acc.count(x) == recount


def test_concurrent_queries_match_serial(rng):
    X = gaussian(rng, 400, 12)
    index = mrpt.grow_trees(X, 8, 4, seed=33)
    Q = gaussian(rng, 40, 12)
    serial = [mrpt.approximate_knn(q, 5, index, votes=2).indices.tolist() for q in Q]
    with ThreadPoolExecutor(max_workers=4) as pool:
        par = list(pool.map(lambda q: mrpt.approximate_knn(q, 5, index, 2).indices.tolist(), Q))
    assert serial == par
    ids, _, _ = mrpt.approximate_knn_batch(Q, 5, index, 2)
    assert [row[row >= 0].tolist() for row in ids] == serial


# --- projection (test_core.py:83-166, test_kernels.py:26-47) --------------------
def test_projection_contract(rng):
    R = _matrix([[2.0], [3.0]])
    assert np.array_equal(mrpt.project_dataset(np.eye(2, dtype=np.float32), R),
                          np.array([[2.0], [3.0]], np.float32))
    R = mrpt.sample_sparse_matrix(4, 2, a=0.8, seed=1)
    assert not mrpt.project_dataset(np.zeros((3, 4), np.float32), R).any()
    R = mrpt.sample_sparse_matrix(30, 5, a=0.4, seed=21)
    X = gaussian(rng, 40, 30)
    P = mrpt.project_dataset(X, R)
    for i in (0, 7, 39):
        assert np.array_equal(mrpt.project_query(X[i], R), P[i])
    with pytest.raises(mrpt.ShapeError):
        mrpt.project_dataset(gaussian(rng, 5, 7), mrpt.sample_sparse_matrix(6, 3, 0.6, seed=8))


def test_mac_counts_fixed_count(rng):
    """test_acceptance.py:200-214 / test_core.py:227-236."""
    d, depth, a = 64, 4, 0.125
    X = gaussian(rng, 256, d)
    per = math.ceil(a * d)
    with mrpt.count_macs() as c:
        index = mrpt.grow_trees(X, 3, depth, a, seed=8, fixed_count=True)
    assert c.macs == 3 * per * depth * 256
    with mrpt.count_macs() as c:
        mrpt.approximate_knn(gaussian(rng, 1, d)[0], 5, index, votes=1)
    assert c.macs == 3 * per * depth


def test_dataset_device_and_checksum(rng):
    import torch

    X = gaussian(rng, 10, 4)
    a = mrpt.Dataset(X)
    b = mrpt.Dataset(torch.from_numpy(X).cuda())
    assert a.checksum == b.checksum == O.fnv1a64(X.tobytes())
    assert a.checksum != mrpt.Dataset(gaussian(rng, 10, 4)).checksum
    with pytest.raises(mrpt.ParameterError):
        mrpt.Dataset(torch.tensor([[1.0, float("nan")]], device="cuda"))


def test_recall_monotone_in_votes():
    """test_acceptance.py:156-174: mean recall non-increasing over v."""
    rng = np.random.default_rng(505)
    X = gaussian(rng, 5000, 50)
    Q = gaussian(rng, 100, 50)
    index = mrpt.grow_trees(X, 20, 6, seed=99)
    truth = np.stack([O.brute_force_knn(X, q, 10)[0] for q in Q])
    means = []
    for v in range(1, 6):
        ids, _, _ = mrpt.approximate_knn_batch(Q, 10, index, v)
        means.append(np.mean([len(np.intersect1d(a[a >= 0], b)) / 10 for a, b in zip(ids, truth)]))
    assert all(means[i] >= means[i + 1] for i in range(len(means) - 1))
