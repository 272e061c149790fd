"""Generate golden fixtures from the UNMODIFIED reference package.

Run in the build container (where /root/reference exists):

    ./oracle/build_ref.sh && python tests/golden/make_golden.py

It imports the reference's ``mrpt`` from oracle/_ref (compiled backend) and
records, for a set of small seeded cases plus the full BASELINE config 1,
the reference's own outputs: sparse matrices, split values, leaf offsets and
leaf ids (grow_trees, trees.py:187-245), per-query leaves (_route_all,
search.py:116-120), candidate sets (candidate_set, search.py:130-143) and
k-NN answers (approximate_knn, search.py:175-184), FNV-1a checksums
(_cy.pyx:100-106).  The .npz files are committed; nothing at test time reads
/root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
sys.path.insert(0, ROOT)

import mrpt  # noqa: E402  (the reference)
from mrpt import _kernels  # noqa: E402
from mrpt.search import _route_all  # noqa: E402

from paper_1509_06957_b200 import workloads  # noqa: E402

assert _kernels.backend() == "compiled"


def pack_index(index):
    mats = index.matrices
    nnz = np.array([R.nnz for R in mats], dtype=np.int64)
    return dict(
        mat_nnz=nnz,
        mat_col_ptr=np.stack([R.col_ptr for R in mats]),
        mat_rows=np.concatenate([R.row_idx for R in mats]) if nnz.sum() else np.zeros(0, np.int32),
        mat_vals=np.concatenate([R.values for R in mats]) if nnz.sum() else np.zeros(0, np.float32),
        splits=index.splits, leaf_offsets=index.leaf_offsets, leaf_indices=index.leaf_indices,
        checksum=np.uint64(index.dataset_checksum),
    )


def query_block(index, Q, k, votes, sets_for=None):
    out = {}
    leaves = np.stack([_route_all(np.ascontiguousarray(q), index) for q in Q])
    out["leaves"] = leaves.astype(np.int32)
    for v in votes:
        ids = np.full((len(Q), k), -1, dtype=np.int64)
        dists = np.full((len(Q), k), np.inf)
        counts = np.zeros(len(Q), dtype=np.int64)
        for i, q in enumerate(Q):
            r = mrpt.approximate_knn(q, k, index, votes=v)
            ids[i, :len(r)] = r.indices
            dists[i, :len(r)] = r.distances
            counts[i] = r.candidate_count
        out[f"ids_v{v}"] = ids
        out[f"dists_v{v}"] = dists
        out[f"counts_v{v}"] = counts
        ns = len(Q) if sets_for is None else min(sets_for, len(Q))
        sets, bounds = [], [0]
        for i in range(ns):
            c, _ = mrpt.candidate_set(Q[i], index, v)
            c = np.sort(c)
            sets.append(c)
            bounds.append(bounds[-1] + len(c))
        out[f"cand_v{v}"] = np.concatenate(sets).astype(np.int32) if sets else np.zeros(0, np.int32)
        out[f"cand_bounds_v{v}"] = np.array(bounds, dtype=np.int64)
    return out


SMALL = [
    # name, generator, n, d, T, depth, sparsity, seed, fixed_count, nq, k, votes
    ("gauss_400x24", "gauss", 400, 24, 6, 4, None, 13, False, 40, 8, (1, 2, 3)),
    ("gauss_300x10", "gauss", 300, 10, 6, 3, None, 14, False, 30, 5, (1, 2, 6)),
    ("duplicates_16x4", "ones", 16, 4, 2, 3, None, 1, False, 6, 4, (1, 2)),
    ("int_ties_2000x16", "ints", 2000, 16, 4, 6, None, 5, False, 30, 10, (1, 2, 4)),
    ("sparse_zero_cols_500x8", "gauss", 500, 8, 6, 5, 0.05, 3, False, 30, 6, (1, 3)),
    ("fixed_count_256x64", "gauss", 256, 64, 3, 4, 0.125, 8, True, 20, 5, (1, 2)),
    ("full_depth_8x5", "gauss", 8, 5, 2, 3, 1.0, 11, False, 4, 3, (1, 2)),
    ("odd_1001x33", "gauss", 1001, 33, 5, 7, None, 21, False, 40, 12, (1, 2, 5)),
    ("clustered_3000x96", "clusters", 3000, 96, 12, 6, None, 99, False, 50, 10, (1, 2, 4)),
]


def make_data(kind, n, d, rng):
    if kind == "gauss":
        return rng.standard_normal((n, d)).astype(np.float32)
    if kind == "ones":
        return np.ones((n, d), dtype=np.float32)
    if kind == "ints":
        return rng.integers(0, 4, size=(n, d)).astype(np.float32)
    if kind == "clusters":
        c = 4.0 * rng.standard_normal((10, d))
        return (c[rng.integers(0, 10, size=n)] + rng.standard_normal((n, d))).astype(np.float32)
    raise KeyError(kind)


def main():
    rng = np.random.default_rng(20240817)
    # FNV-1a: the reference test vectors (pkg/tests/test_io.py:177-186) + random buffers
    bufs = [b"", b"a", b"foobar"] + [rng.integers(0, 256, size=s).astype(np.uint8).tobytes()
                                     for s in (1, 7, 1024, 4099, 65537)]
    blob = b"".join(bufs)
    lens = np.array([len(b) for b in bufs], dtype=np.int64)
    hashes = np.array([_kernels.fnv1a64(np.frombuffer(b, dtype=np.uint8)) for b in bufs],
                      dtype=np.uint64)
    np.savez_compressed(os.path.join(HERE, "fnv.npz"), blob=np.frombuffer(blob, dtype=np.uint8),
                        lens=lens, hashes=hashes)

    for (name, kind, n, d, T, depth, a, seed, fixed, nq, k, votes) in SMALL:
        X = make_data(kind, n + nq, d, rng)
        Xd, Q = X[:n], X[n:]
        if kind == "ones":
            Q = np.stack([np.full(d, s, np.float32) for s in (3.0, -3.0, 0.0, 1.0, 2.0, -1.0)])
        index = mrpt.grow_trees(Xd, n_trees=T, depth=depth, sparsity=a, seed=seed,
                                fixed_count=fixed)
        rec = dict(X=Xd, Q=Q, n_trees=T, depth=depth,
                   sparsity=np.float64(index.sparsity), seed=seed, fixed_count=fixed, k=k,
                   votes=np.array(votes))
        rec.update(pack_index(index))
        rec.update(query_block(index, Q, k, votes))
        np.savez_compressed(os.path.join(HERE, f"small_{name}.npz"), **rec)
        print("wrote", name, file=sys.stderr)

    # a reference-written index file (persistence.py:33-58), for byte-level checks
    g = np.load(os.path.join(HERE, "small_gauss_400x24.npz"))
    idx = mrpt.grow_trees(g["X"], n_trees=int(g["n_trees"]), depth=int(g["depth"]),
                          seed=int(g["seed"]))
    mrpt.save_index(idx, os.path.join(HERE, "index_gauss_400x24.mrpt"))

    # full BASELINE config 1 (regenerated from the pinned generator at test time)
    X, Q, p = workloads.generate(1)
    index = mrpt.grow_trees(X, p["n_trees"], p["depth"], p["sparsity"], seed=p["seed"])
    rec = dict(x_checksum=np.uint64(_kernels.fnv1a64(X.view(np.uint8).reshape(-1))),
               q_checksum=np.uint64(_kernels.fnv1a64(Q.view(np.uint8).reshape(-1))),
               n_trees=p["n_trees"], depth=p["depth"], sparsity=np.float64(p["sparsity"]),
               seed=p["seed"], k=p["k"], votes=np.array((1, 2)))
    rec.update(pack_index(index))
    rec.update(query_block(index, Q, p["k"], (1, 2), sets_for=25))
    np.savez_compressed(os.path.join(HERE, "config1.npz"), **rec)
    print("wrote config1", file=sys.stderr)
    with open(os.path.join(HERE, "NUMPY_VERSION"), "w") as fh:
        fh.write(np.__version__ + "\n")


if __name__ == "__main__":
    main()
