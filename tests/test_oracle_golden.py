"""Pin the CPU oracle against the reference's own outputs (tests/golden/*.npz,
produced by the unmodified reference via tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import golden, golden_small_names, unpack_matrices
from oracle import oracle as O
from paper_1509_06957_b200 import workloads


def _index_from_golden(g):
    mats = unpack_matrices(g)
    return dict(matrices=mats, splits=g["splits"], leaf_offsets=g["leaf_offsets"],
                leaf_indices=g["leaf_indices"], depth=int(g["depth"]))


def test_fnv_known_vectors():
    g = golden("fnv.npz")
    blob = g["blob"].tobytes()
    off = 0
    for ln, h in zip(g["lens"], g["hashes"]):
        assert O.fnv1a64(blob[off:off + int(ln)]) == int(h)
        off += int(ln)
    # the reference's own known answers (pkg/tests/test_io.py:177-186)
    assert O.fnv1a64(b"") == 0xCBF29CE484222325
    assert O.fnv1a64(b"a") == 0xAF63DC4C8601EC8C
    assert O.fnv1a64(b"foobar") == 0x85944171F73967E8


@pytest.mark.parametrize("name", golden_small_names())
def test_oracle_build_matches_reference(name):
    g = golden(name)
    built = O.grow_trees(g["X"], int(g["n_trees"]), int(g["depth"]), float(g["sparsity"]),
                         int(g["seed"]), bool(g["fixed_count"]))
    for (cp, r, v), (gcp, gr, gv) in zip(built["matrices"], unpack_matrices(g)):
        assert np.array_equal(cp, gcp) and np.array_equal(r, gr)
        assert v.tobytes() == gv.tobytes()
    assert built["splits"].tobytes() == g["splits"].tobytes()
    assert np.array_equal(built["leaf_offsets"], g["leaf_offsets"])
    assert np.array_equal(built["leaf_indices"], g["leaf_indices"])
    assert O.fnv1a64(g["X"].tobytes()) == int(g["checksum"])


@pytest.mark.parametrize("name", golden_small_names())
def test_oracle_queries_match_reference(name):
    g = golden(name)
    idx = _index_from_golden(g)
    leaves = O.query_leaves(g["Q"], idx)
    assert np.array_equal(leaves, g["leaves"])
    for v in g["votes"]:
        b = g[f"cand_bounds_v{v}"]
        for i in range(len(b) - 1):
            assert np.array_equal(O.candidates(leaves[i], idx, int(v)),
                                  g[f"cand_v{v}"][b[i]:b[i + 1]])
        ids, dists, counts = O.approximate_knn_batch(g["X"], g["Q"], int(g["k"]), idx, int(v))
        assert np.array_equal(ids, g[f"ids_v{v}"])
        assert np.array_equal(counts, g[f"counts_v{v}"])
        np.testing.assert_allclose(dists, g[f"dists_v{v}"], rtol=1e-12)


def test_oracle_config1_matches_reference():
    g = golden("config1.npz")
    X, Q, p = workloads.generate(1)
    assert O.fnv1a64(X.tobytes()) == int(g["x_checksum"]), "config-1 generator drifted"
    assert O.fnv1a64(Q.tobytes()) == int(g["q_checksum"])
    built = O.grow_trees(X, int(g["n_trees"]), int(g["depth"]), float(g["sparsity"]),
                         int(g["seed"]))
    assert built["splits"].tobytes() == g["splits"].tobytes()
    assert np.array_equal(built["leaf_offsets"], g["leaf_offsets"])
    assert np.array_equal(built["leaf_indices"], g["leaf_indices"])
    leaves = O.query_leaves(Q, built)
    assert np.array_equal(leaves, g["leaves"])
    ids, dists, counts = O.approximate_knn_batch(X, Q[:200], int(g["k"]), built, 2)
    assert np.array_equal(ids, g["ids_v2"][:200])
    assert np.array_equal(counts, g["counts_v2"][:200])
    np.testing.assert_allclose(dists, g["dists_v2"][:200], rtol=1e-12)


# --- ground truth (f3) and the compiled vote order -----------------------------
@pytest.mark.parametrize("d", [1, 5, 7, 8, 9, 24, 100, 128, 129, 200, 256, 384, 784, 960, 1000, 4096])
def test_pairwise_plan_is_numpys_sum(d):
    """The restated summation plan (what the GPU ground-truth kernel runs)
    equals numpy's own row sum -- the reference's d2 (evaluation.py:40-41)."""
    rng = np.random.default_rng(d)
    diff = rng.standard_normal((20, d))
    sq = diff * diff
    want = sq.sum(axis=1)
    got = np.array([O.pairwise_sum(r) for r in sq])
    assert got.tobytes() == want.tobytes()


def test_oracle_ground_truth_matches_reference():
    g = golden("ground_truth.npz")
    for name in g["names"]:
        X, Q, k = g[f"{name}_X"], g[f"{name}_Q"], int(g[f"{name}_k"])
        ids, dists = O.compute_ground_truth(X, Q, k)
        assert np.array_equal(ids, g[f"{name}_ids"]), name
        assert dists.tobytes() == g[f"{name}_dists"].tobytes(), name
    ids, dists, n = O.brute_force_knn(g["kgtn_X"], g["kgtn_q"], 20)
    assert n == 9 and np.array_equal(ids, g["kgtn_ids"])
    assert dists.tobytes() == g["kgtn_dists"].tobytes()


def test_oracle_crossing_order_matches_compiled_reference():
    g = golden("candidates_unsorted.npz")
    idx = O.grow_trees(g["X"], int(g["n_trees"]), int(g["depth"]), seed=int(g["seed"]))
    leaves = O.query_leaves(g["Q"], idx)
    b = g["bounds"]
    i = 0
    for v in g["votes"]:
        for qi in range(len(g["Q"])):
            got = O.candidates_crossing_order(leaves[qi], idx, int(v))
            assert np.array_equal(got, g["cand"][b[i]:b[i + 1]])
            i += 1
