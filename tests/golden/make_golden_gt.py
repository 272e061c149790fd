"""Golden fixtures for ground truth (f3) and the compiled vote order, from the
UNMODIFIED reference package.

Run in the build container (where /root/reference exists):

    ./oracle/build_ref.sh && python tests/golden/make_golden_gt.py

Writes ``ground_truth.npz``: for seeded cases (Gaussian, exact duplicates,
integer data with distance ties, k > n, widths below 8, above 128 and the
BASELINE widths 784 / 960 that exercise numpy's pairwise-summation split) the
reference's ``compute_ground_truth`` (evaluation.py:65-81) and
``brute_force_knn`` (evaluation.py:28-47) outputs; and
``candidates_unsorted.npz``: the compiled backend's candidate lists in its
own threshold-crossing order (``candidate_set``, search.py:130-143 ->
_cy.vote), unsorted.  Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))

import mrpt  # noqa: E402  (the reference)
from mrpt import _kernels  # noqa: E402
from mrpt.evaluation import brute_force_knn, compute_ground_truth  # noqa: E402

assert _kernels.backend() == "compiled"

# name, kind, n, d, nq, k
CASES = [
    ("gauss_500x24", "gauss", 500, 24, 30, 10),
    ("dups_64x16", "dups", 64, 16, 8, 12),
    ("int_ties_700x9", "ints", 700, 9, 20, 25),
    ("narrow_300x5", "gauss", 300, 5, 10, 7),
    ("wide_400x784", "unit", 400, 784, 12, 10),
    ("wide_300x960", "unit", 300, 960, 8, 100),
    ("odd_1500x200", "gauss", 1500, 200, 16, 600),
]


def make(kind, n, d, rng):
    if kind == "gauss":
        return rng.standard_normal((n, d)).astype(np.float32)
    if kind == "dups":  # every row appears 4 times: exact distance ties
        base = rng.standard_normal((n // 4, d)).astype(np.float32)
        return np.repeat(base, 4, axis=0)
    if kind == "ints":
        return rng.integers(0, 3, size=(n, d)).astype(np.float32)
    if kind == "unit":
        return rng.random((n, d)).astype(np.float32)
    raise KeyError(kind)


def main():
    rng = np.random.default_rng(5150)
    rec = {}
    for name, kind, n, d, nq, k in CASES:
        allx = make(kind, n + nq, d, rng)
        X, Q = allx[:n], allx[n:]
        if kind == "dups":
            Q = X[::5][:nq] + 0.0  # queries on top of duplicated rows
        gt = compute_ground_truth(X, Q, k)
        rec[f"{name}_X"] = X
        rec[f"{name}_Q"] = Q
        rec[f"{name}_k"] = np.int64(k)
        rec[f"{name}_ids"] = gt.indices
        rec[f"{name}_dists"] = gt.distances
    # k > n through brute_force_knn: min(k, n) neighbours
    X = rng.standard_normal((9, 6)).astype(np.float32)
    q = rng.standard_normal(6)  # float64 query: the reference keeps it float64
    r = brute_force_knn(q, 20, X)
    rec.update(kgtn_X=X, kgtn_q=q, kgtn_ids=r.indices, kgtn_dists=r.distances)
    np.savez_compressed(os.path.join(HERE, "ground_truth.npz"), names=np.array([c[0] for c in CASES]),
                        **rec)

    # compiled-order candidate lists
    c = 4.0 * rng.standard_normal((12, 32))
    allx = (c[rng.integers(0, 12, size=2040)] + rng.standard_normal((2040, 32))).astype(np.float32)
    X, Q = allx[:2000], allx[2000:]
    index = mrpt.grow_trees(X, n_trees=10, depth=5, seed=77)
    lists, bounds = [], [0]
    for v in (1, 2, 3):
        for q in Q:
            cand, _ = mrpt.candidate_set(q, index, v)
            lists.append(np.asarray(cand, dtype=np.int64))
            bounds.append(bounds[-1] + len(cand))
    np.savez_compressed(os.path.join(HERE, "candidates_unsorted.npz"), X=X, Q=Q, n_trees=10, depth=5,
                        seed=77, votes=np.array((1, 2, 3)), cand=np.concatenate(lists),
                        bounds=np.array(bounds, dtype=np.int64))
    print("wrote ground_truth.npz, candidates_unsorted.npz", file=sys.stderr)


if __name__ == "__main__":
    main()
