"""Host-side API behaviour that needs no GPU: validation order and error
types match the reference (pkg/src/mrpt/core.py, trees.py, search.py), and
host-side sampling is bit-identical to the reference's."""

import math

import numpy as np
import pytest

import paper_1509_06957_b200 as mrpt
from conftest import gaussian, golden, golden_small_names, unpack_matrices


def test_sample_sparse_matrix_matches_reference_streams():
    for name in golden_small_names():
        g = golden(name)
        d = g["X"].shape[1]
        for t, (cp, r, v) in enumerate(unpack_matrices(g)):
            R = mrpt.sample_sparse_matrix(d, int(g["depth"]), float(g["sparsity"]),
                                          seed=(int(g["seed"]), t),
                                          fixed_count=bool(g["fixed_count"]))
            assert np.array_equal(R.col_ptr, cp) and np.array_equal(R.row_idx, r)
            assert R.values.tobytes() == v.tobytes()


@pytest.mark.parametrize("bad_a", [1.5, 0.0, -0.25])
def test_sparsity_out_of_range_rejected(bad_a):
    with pytest.raises(mrpt.ParameterError):
        mrpt.sample_sparse_matrix(4, 2, a=bad_a, seed=5)


@pytest.mark.parametrize("d,depth", [(0, 2), (4, 0)])
def test_degenerate_shape_rejected(d, depth):
    with pytest.raises(mrpt.ParameterError):
        mrpt.sample_sparse_matrix(d, depth, a=0.5, seed=5)


def test_bad_seed_rejected():
    with pytest.raises(mrpt.ParameterError):
        mrpt.sample_sparse_matrix(4, 2, a=0.5, seed=-1)
    with pytest.raises(mrpt.ParameterError):
        mrpt.sample_sparse_matrix(4, 2, a=0.5, seed=(1, "x"))


def test_fixed_count_columns():
    R = mrpt.sample_sparse_matrix(37, 5, 0.21, seed=3, fixed_count=True)
    assert (R.nonzeros_per_column() == math.ceil(0.21 * 37)).all()
    for j in range(5):
        assert (np.diff(R.row_idx[R.col_ptr[j]:R.col_ptr[j + 1]]) > 0).all()


def test_dataset_validation_on_host():
    with pytest.raises(mrpt.ParameterError):
        mrpt.Dataset(np.array([[1.0, np.nan]], dtype=np.float32))
    with pytest.raises(mrpt.ParameterError):
        mrpt.Dataset(np.array([[np.inf, 1.0]], dtype=np.float32))
    with pytest.raises(mrpt.ParameterError):
        mrpt.Dataset(np.empty((0, 3), dtype=np.float32))
    with pytest.raises(mrpt.ShapeError):
        mrpt.Dataset(np.zeros(4, dtype=np.float32))
    X = mrpt.Dataset(np.ones((3, 3)))
    assert X.values.dtype == np.float32 and not X.values.flags.writeable


def test_grow_trees_validation_precedes_device_work(rng):
    X = gaussian(rng, 8, 5)
    with pytest.raises(mrpt.ParameterError):
        mrpt.grow_trees(X, n_trees=0, depth=2, seed=0)
    with pytest.raises(mrpt.DepthError):
        mrpt.grow_trees(X, n_trees=1, depth=4, seed=0)
    with pytest.raises(mrpt.DepthError):
        mrpt.grow_trees(X, n_trees=1, depth=0, seed=0)
    with pytest.raises(mrpt.ParameterError):
        mrpt.grow_trees(X, n_trees=1, depth=2, seed=-1)
    with pytest.raises(mrpt.ParameterError):
        mrpt.grow_trees(X, n_trees=1, depth=2, threads=0)


def test_median_split_and_exact_scan_argument_errors():
    with pytest.raises(mrpt.ParameterError):
        mrpt.median_split(np.array([1.0]), np.array([0]))
    with pytest.raises(mrpt.ParameterError):
        mrpt.exact_knn_in_set(np.zeros(3), 0, np.arange(2), np.zeros((4, 3)))
    with pytest.raises(mrpt.ShapeError):
        mrpt.exact_knn_in_set(np.zeros(2), 1, np.arange(2), np.zeros((4, 3)))


def test_euclidean_distance_host_helper():
    assert mrpt.euclidean_distance([0.0, 0.0], [3.0, 4.0]) == 5.0
    with pytest.raises(mrpt.ShapeError):
        mrpt.euclidean_distance([1.0, 2.0], [1.0, 2.0, 3.0])


def test_mac_counter_nesting():
    from paper_1509_06957_b200.core import _record_macs

    with mrpt.count_macs() as outer:
        _record_macs(5)
        with mrpt.count_macs() as inner:
            _record_macs(7)
    assert outer.macs == 12 and inner.macs == 7


def test_workload_generators_are_deterministic():
    from paper_1509_06957_b200 import workloads

    for c in (1, 2, 3, 4, 5):
        X1, Q1, p = workloads.generate(c, scale=0.0002 if c > 1 else 0.05)
        X2, Q2, _ = workloads.generate(c, scale=0.0002 if c > 1 else 0.05)
        assert X1.dtype == np.float32 and X1.shape[1] == p["d"]
        assert np.array_equal(X1, X2) and np.array_equal(Q1, Q2)
        assert 2 ** p["depth"] <= X1.shape[0]


@pytest.mark.parametrize("nq", [4096, 4097, 5000, 10000, 10001, 65536])
@pytest.mark.parametrize("mode", ["", "equal"])
def test_pipelined_piece_bounds_partition_the_batch(nq, mode):
    """The overlapped host path cuts a batch into ascending pieces that cover
    every query exactly once, with a small first piece by default."""
    from paper_1509_06957_b200.search import _pipe_bounds

    b = _pipe_bounds(nq, mode)
    assert b[0] == 0 and b[-1] == nq
    assert all(x < y for x, y in zip(b, b[1:]))
    assert 1 <= len(b) - 1 <= 4
    if mode == "":
        assert b[1] - b[0] <= max(256, nq // 8)


class _FakeRows:
    def __init__(self, stride):
        self._s = stride

    def stride(self, i):
        return self._s

    def data_ptr(self):
        return 1 << 20


class _FakeIndex:
    def __init__(self, n, d, u8=True, fp16=False, stride=None):
        self.n, self.d = n, d
        self.X = _FakeRows(stride if stride is not None else d)
        self._u8, self._h = u8, fp16

    def u8_rows(self):
        # (rows, row stride, ...): the stride is the shadow width round_up(d, 16)
        return (None, (self.d + 15) // 16 * 16) if self._u8 else None

    def shadow(self):
        return object() if self._h else None



@pytest.mark.parametrize("n,d,k,u8,want", [
    (60_000, 784, 10, True, ["u8", "u8tc_bits", "fp32"]),
    (60_000, 784, 17, True, ["u8", "fp32"]),                # tcgen05 filter: k <= 16
    (60_000, 1000, 10, True, ["u8", "u8tc_bits", "fp32"]),  # ldq 1008
    (60_000, 100, 10, True, ["u8", "fp32"]),                # tcgen05 filter: ldq >= 128
    (60_000, 37, 10, True, ["u8", "fp32"]),                 # no 16-byte rows
    (5_000_000, 128, 10, True, ["u8", "fp32"]),             # bitmaps of at most 4M ids
    (60_000, 784, 121, True, ["fp32"]),                     # filters take k <= 120
    (60_000, 784, 10, False, ["fp32"]),                     # signed data: no u8 shadow
])
def test_scan_route_availability(n, d, k, u8, want):
    from paper_1509_06957_b200.search import _scan_variants

    assert _scan_variants(_FakeIndex(n, d, u8), k) == want


def test_build_batches_are_equal_sized():
    """Trees per K1+K5 batch: as many as memory allows, but in equal batches
    (no small last batch): config 5's 1000 trees go as 10 x 100, not 9 x 111 + 1."""
    from paper_1509_06957_b200.trees import _batch_trees

    n, d, depth, T = 10_000_000, 256, 13, 1000
    per_tree = n * (4 * depth + 8) + 3 * n + (1 << 20)
    tb = _batch_trees(n, d, depth, T, free_bytes=2 * 111 * per_tree)
    assert tb == 100
    assert _batch_trees(n, d, depth, 7, free_bytes=2 * 111 * per_tree) == 7
    assert _batch_trees(n, d, depth, T, free_bytes=per_tree) == 1
    for free_trees in (3, 17, 64, 200):
        tb = _batch_trees(n, d, depth, T, free_bytes=2 * free_trees * per_tree)
        nb = -(-T // tb)
        assert tb <= min(free_trees, 128) and nb * tb - T < nb  # batches differ by at most one tree
