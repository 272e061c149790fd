"""Index files: byte-identical to the reference's writer, loadable from it, and
the reference's corruption checks (pkg/tests/test_io.py:103-171)."""

import os

import numpy as np
import pytest

import paper_1509_06957_b200 as mrpt
from conftest import GOLDEN, gaussian, golden

pytestmark = pytest.mark.gpu

REF_FILE = os.path.join(GOLDEN, "index_gauss_400x24.mrpt")


def test_save_is_byte_identical_to_reference(tmp_path):
    g = golden("small_gauss_400x24.npz")
    index = mrpt.grow_trees(g["X"], int(g["n_trees"]), int(g["depth"]), seed=int(g["seed"]))
    out = tmp_path / "ours.mrpt"
    mrpt.save_index(index, out)
    assert out.read_bytes() == open(REF_FILE, "rb").read()


def test_reference_file_loads_and_answers_identically():
    g = golden("small_gauss_400x24.npz")
    loaded = mrpt.load_index(REF_FILE, g["X"])
    assert loaded.splits.tobytes() == g["splits"].tobytes()
    for v in g["votes"]:
        ids, dists, counts = mrpt.approximate_knn_batch(g["Q"], int(g["k"]), loaded, int(v))
        assert np.array_equal(ids, g[f"ids_v{int(v)}"])
        assert np.array_equal(counts.astype(np.int64), g[f"counts_v{int(v)}"])


def test_round_trip_and_flags(rng, tmp_path):
    X = mrpt.Dataset(gaussian(rng, 600, 24))
    a = mrpt.grow_trees(X, 5, 4, seed=2024)
    p1, p2 = tmp_path / "a.mrpt", tmp_path / "b.mrpt"
    mrpt.save_index(a, p1)
    mrpt.save_index(mrpt.grow_trees(X, 5, 4, seed=2024), p2)
    assert p1.read_bytes() == p2.read_bytes()
    b = mrpt.load_index(p1, X)
    Q = gaussian(rng, 30, 24)
    for r1, r2 in zip(mrpt.approximate_knn_batch(Q, 8, a, 2), mrpt.approximate_knn_batch(Q, 8, b, 2)):
        assert np.array_equal(r1, r2)
    fc = mrpt.grow_trees(mrpt.Dataset(gaussian(rng, 64, 16)), 2, 3, sparsity=0.25, seed=9,
                         fixed_count=True)
    mrpt.save_index(fc, tmp_path / "fc.mrpt")
    assert mrpt.load_index(tmp_path / "fc.mrpt", fc.dataset).fixed_count is True


def test_corruption_is_rejected(rng, tmp_path):
    g = golden("small_gauss_400x24.npz")
    blob = open(REF_FILE, "rb").read()
    with pytest.raises(mrpt.ChecksumMismatchError):
        mrpt.load_index(REF_FILE, gaussian(rng, 400, 24))
    cases = {
        "truncated": blob[:-7],
        "trailing": blob + b"\0",
        "magic": b"XXXXXXXX" + blob[8:],
        "version": blob[:8] + (2).to_bytes(4, "little") + blob[12:],
        "header": blob[:20],
    }
    for name, data in cases.items():
        p = tmp_path / f"{name}.mrpt"
        p.write_bytes(data)
        with pytest.raises(mrpt.FormatError):
            mrpt.load_index(p, g["X"])
