"""Parity at the BASELINE configurations ("no reference test
exercises the BASELINE configs; at that scale parity is differential").

* Config 2 (n=60k, d=784, T=100): the whole index is rebuilt by the oracle
  and compared bit for bit; all 10,000 queries at v=2 and 1,000 at v=1 (the
  fused tcgen05 filter route) through the oracle's approximate_knn_batch.
* Configs 3-5 (n = 1M / 1M / 10M): sampled trees rebuilt by the oracle
  (O.build_one_tree, trees.py:217-224 -- every tree is i.i.d. in (seed, t)),
  and queries answered by the oracle over the GPU-built index (the leaf
  slices each query lands in are read back from the device; the vote,
  candidate set and exact float64 scan are the oracle's).

Counts, neighbour ids and float64 distance bytes must be identical; the
report also prints how often the exact fallbacks fired.  Data come from
paper_1509_06957_b200.workloads (seeded synthetic stand-ins)."""

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import paper_1509_06957_b200 as mrpt
from oracle import oracle as O
from paper_1509_06957_b200 import workloads
from paper_1509_06957_b200.search import _route_device, fallback_stats

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _device_build(X, p):
    import torch

    return mrpt.grow_trees(torch.from_numpy(X).cuda(), p["n_trees"], p["depth"], p["sparsity"],
                           seed=p["seed"])


def _check_trees(X, p, index, ts):
    D = index.device_index()

    def one(t):
        R, (s_, o_, i_) = O.build_one_tree(X, p["depth"], p["sparsity"], p["seed"], t)
        return (R[2].tobytes() == index.matrices[t].values.tobytes()
                and s_.tobytes() == D.splits[t].cpu().numpy().tobytes()
                and np.array_equal(o_, D.offsets[t].cpu().numpy())
                and np.array_equal(i_, D.indices[t].cpu().numpy()))

    with ThreadPoolExecutor(len(ts)) as ex:
        ok = list(ex.map(one, ts))
    assert all(ok), [t for t, g in zip(ts, ok) if not g]


def _oracle_over_device_index(X, Q, index, k, v):
    """approximate_knn (search.py:175-184) per query, restated by the oracle,
    over the GPU-built index: leaves by the oracle's own projection + descent
    (splits and matrices from the index), the leaf slices read from the
    device, counts by exact bincount, the oracle's exact scan."""
    import torch

    D = index.device_index()
    ref = dict(matrices=[(R.col_ptr, R.row_idx, R.values) for R in index.matrices],
               splits=D.splits.cpu().numpy(), depth=index.depth)
    leaves = O.query_leaves(Q, ref)
    # the GPU's own route must agree
    assert np.array_equal(_route_device(torch.from_numpy(Q).cuda(), D).cpu().numpy(), leaves)
    offs = D.offsets.cpu().numpy()
    flat = D.indices.view(-1)
    T, n = index.n_trees, X.shape[0]
    ids = np.full((len(Q), k), -1, np.int64)
    dists = np.full((len(Q), k), np.inf)
    counts = np.zeros(len(Q), np.int64)
    tr = np.arange(T)
    for i in range(len(Q)):
        s0 = offs[tr, leaves[i]]
        lens = offs[tr, leaves[i] + 1] - s0
        # every occurrence of every id of the T leaf slices: element j of the
        # concatenation sits at t*n + s0[t] + (j - first rank of slice t)
        base = tr * n + s0 - (np.cumsum(lens) - lens)
        idx = np.repeat(base, lens) + np.arange(int(lens.sum()))
        allids = flat[torch.from_numpy(idx).cuda()].cpu().numpy()
        c = np.bincount(allids, minlength=X.shape[0])
        S = np.flatnonzero(c >= v)
        a, b, m = O.exact_knn(X, Q[i], k, S)
        ids[i, :len(a)] = a
        dists[i, :len(b)] = b
        counts[i] = m
    return ids, dists, counts


def _compare(got, want):
    ids, dists, counts = got
    rids, rd, rc = want
    assert np.array_equal(counts.astype(np.int64), rc)
    assert np.array_equal(ids, rids)
    assert dists.tobytes() == rd.tobytes()


def test_config2_full_index_and_queries():
    X, Q, p = workloads.generate(2)
    index = _device_build(X, p)
    ref = O.grow_trees(X, p["n_trees"], p["depth"], p["sparsity"], p["seed"])
    D = index.device_index()
    assert D.splits.cpu().numpy().tobytes() == ref["splits"].tobytes()
    assert np.array_equal(D.offsets.cpu().numpy(), ref["leaf_offsets"])
    assert np.array_equal(D.indices.cpu().numpy(), ref["leaf_indices"])
    fallback_stats(reset=True)
    for v, nq in ((2, 10_000), (1, 1000)):
        got = mrpt.approximate_knn_batch(Q[:nq], p["k"], index, v)
        _compare(got, O.approximate_knn_batch(X, Q[:nq], p["k"], ref, v))
    print("config 2 fallbacks:", fallback_stats())


# >= 256 queries: the per-index route autotune runs, so the batches go
# through the routes the bench uses at these sizes (fp16 at configs 4-5)
@pytest.mark.parametrize("config,votes,nq,trees", [(3, (2, 4), 1000, 4), (4, (10, 5), 1000, 4),
                                                   (5, (10,), 300, 4)])
def test_large_config_sampled_trees_and_queries(config, votes, nq, trees):
    X, Q, p = workloads.generate(config)
    index = _device_build(X, p)
    T = p["n_trees"]
    _check_trees(X, p, index, sorted({int(round(x)) for x in np.linspace(0, T - 1, trees)}))
    fallback_stats(reset=True)
    for v in votes:
        got = mrpt.approximate_knn_batch(Q[:nq], p["k"], index, v)
        _compare(got, _oracle_over_device_index(X, Q[:nq], index, p["k"], v))
    print(f"config {config} fallbacks:", fallback_stats())
