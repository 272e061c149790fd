"""GPU parity: the CUDA path against the reference's golden outputs and the
oracle.  Bit-exact for splits, leaf offsets/ids, leaves, candidate sets,
neighbour ids and distances (the kernels reproduce the reference's float64
summation order exactly)."""

import numpy as np
import pytest

import paper_1509_06957_b200 as mrpt
from conftest import gaussian, golden, golden_small_names, unpack_matrices
from oracle import oracle as O
from paper_1509_06957_b200 import workloads
from paper_1509_06957_b200.search import _route_device
from paper_1509_06957_b200 import _device

pytestmark = pytest.mark.gpu


def _check_index(index, g):
    for R, (cp, r, v) in zip(index.matrices, unpack_matrices(g)):
        assert np.array_equal(R.col_ptr, cp) and np.array_equal(R.row_idx, r)
        assert R.values.tobytes() == v.tobytes()
    assert index.splits.tobytes() == g["splits"].tobytes()
    assert np.array_equal(index.leaf_offsets, g["leaf_offsets"])
    assert np.array_equal(index.leaf_indices, g["leaf_indices"])
    assert index.dataset_checksum == int(g["checksum" if "checksum" in g else "x_checksum"])


@pytest.mark.parametrize("name", golden_small_names())
def test_build_and_query_match_reference(name):
    g = golden(name)
    index = mrpt.grow_trees(g["X"], int(g["n_trees"]), int(g["depth"]), float(g["sparsity"]),
                            seed=int(g["seed"]), fixed_count=bool(g["fixed_count"]))
    _check_index(index, g)
    D = index.device_index()
    leaves = _device.d2h(_route_device(_device.h2d(g["Q"]), D))
    assert np.array_equal(leaves, g["leaves"])
    k = int(g["k"])
    for v in g["votes"]:
        v = int(v)
        ids, dists, counts = mrpt.approximate_knn_batch(g["Q"], k, index, v)
        assert np.array_equal(counts.astype(np.int64), g[f"counts_v{v}"])
        assert np.array_equal(ids, g[f"ids_v{v}"])
        assert dists.tobytes() == g[f"dists_v{v}"].tobytes()
        b = g[f"cand_bounds_v{v}"]
        for i in range(min(len(b) - 1, 8)):
            cands, acc = mrpt.candidate_set(g["Q"][i], index, v)
            assert np.array_equal(cands, g[f"cand_v{v}"][b[i]:b[i + 1]])
        r = mrpt.approximate_knn(g["Q"][0], k, index, v)
        assert r.indices.tolist() == g[f"ids_v{v}"][0][:len(r)].tolist()
        assert r.candidate_count == int(g[f"counts_v{v}"][0])


def test_hand_assembled_index_from_golden_arrays():
    """An index assembled from host arrays (as a loaded file would be) queries
    exactly like the reference."""
    g = golden("small_clustered_3000x96.npz")
    mats = [mrpt.SparseProjectionMatrix(d=g["X"].shape[1], depth=int(g["depth"]),
                                        a=float(g["sparsity"]), seed=(int(g["seed"]), t),
                                        col_ptr=cp, row_idx=r, values=v)
            for t, (cp, r, v) in enumerate(unpack_matrices(g))]
    X = mrpt.Dataset(g["X"])
    index = mrpt.MRPTIndex(dataset=X, n_trees=int(g["n_trees"]), depth=int(g["depth"]),
                           sparsity=float(g["sparsity"]), seed=int(g["seed"]), fixed_count=False,
                           matrices=mats, splits=g["splits"], leaf_offsets=g["leaf_offsets"],
                           leaf_indices=g["leaf_indices"], dataset_checksum=int(g["checksum"]))
    for v in g["votes"]:
        ids, dists, counts = mrpt.approximate_knn_batch(g["Q"], int(g["k"]), index, int(v))
        assert np.array_equal(ids, g[f"ids_v{int(v)}"])
        assert np.array_equal(counts.astype(np.int64), g[f"counts_v{int(v)}"])


def test_config1_full_matches_reference():
    g = golden("config1.npz")
    X, Q, p = workloads.generate(1)
    index = mrpt.grow_trees(X, int(g["n_trees"]), int(g["depth"]), float(g["sparsity"]),
                            seed=int(g["seed"]))
    _check_index(index, g)
    for v in (1, 2):
        ids, dists, counts = mrpt.approximate_knn_batch(Q, int(g["k"]), index, v)
        assert np.array_equal(counts.astype(np.int64), g[f"counts_v{v}"])
        assert np.array_equal(ids, g[f"ids_v{v}"])
        assert dists.tobytes() == g[f"dists_v{v}"].tobytes()


# --- kernel-level differential tests against the oracle -----------------------
@pytest.mark.parametrize("ppt", ["2", "4", "8"])
@pytest.mark.parametrize("n,d,depth,a", [(777, 48, 6, 0.25), (3000, 784, 8, 1 / 28),
                                         (200, 1100, 5, 0.05), (5, 3000, 4, 0.01),
                                         (1000, 256, 13, 1 / 16), (2049, 128, 11, 0.09)])
def test_projection_bit_identical(rng, monkeypatch, n, d, depth, a, ppt):
    """K1 with 2, 4 or 8 points per thread is bit-identical to _cy.project."""
    monkeypatch.setenv("MRPT_PROJ_PPT", ppt)
    X = gaussian(rng, n, d)
    R = mrpt.sample_sparse_matrix(d, depth, a, seed=(3, 1))
    P = mrpt.project_dataset(X, R)
    ref = O.project(X, R.col_ptr, R.row_idx, R.values)
    assert P.tobytes() == ref.tobytes()
    for i in (0, n // 2, n - 1):
        assert mrpt.project_query(X[i], R).tobytes() == ref[i].tobytes()


@pytest.mark.parametrize("h32", ["1", "0"])
@pytest.mark.parametrize("n,d,ncols,a", [
    (777, 256, 40, 1 / 16),    # packed tile, 5 points per lane (24 bytes per coordinate), ragged last tile
    (1000, 128, 64, 0.09),     # packed tile at a small d
    (500, 300, 33, 0.05),      # d beyond the 5-point tile: 3 points per lane (16 bytes)
    (333, 440, 35, 0.03),      # the largest 3-point tile rows
    (161, 784, 32, 1 / 28),    # d beyond the packed tiles: plain float64 tile
    (321, 48, 50, 0.25),
])
def test_projection_column_batches_bit_identical(rng, monkeypatch, n, d, ncols, a, h32):
    """K1 on >= 32 columns at once (the build's batches: the float64-tile
    kernels, packed and plain) is bit-identical to _cy.project, including
    zeros, negative zeros, denormals and the largest finite floats."""
    monkeypatch.setenv("MRPT_PROJ_H32", h32)
    X = gaussian(rng, n, d)
    X[::7, ::5] = 0.0
    X[1::11, 3::9] = -0.0
    X[2::13, 1::6] = np.float32(1e-41)      # denormal
    X[3::17, 2::8] = np.float32(-3e-45)     # smallest denormals
    X[4::19, ::10] = np.finfo(np.float32).max
    X[5::23, 4::12] = np.finfo(np.float32).tiny
    R = mrpt.sample_sparse_matrix(d, ncols, a, seed=(5, 2))
    P = mrpt.project_dataset(X, R)
    ref = O.project(X, R.col_ptr, R.row_idx, R.values)
    assert P.tobytes() == ref.tobytes()


@pytest.mark.parametrize("d,T,depth,nq", [
    (256, 70, 9, 1500),    # 5 queries per lane, several tree shares per tile, ragged last tile
    (128, 33, 6, 161),     # forced on a small batch: two tiles, the second of one query
    (400, 40, 7, 1100),    # 3 queries per lane
    (64, 3, 5, 2000),      # fewer trees than warps
])
def test_batched_route_on_packed_tile_matches_oracle(rng, monkeypatch, d, T, depth, nq):
    """K2 on the packed tile (the batched route of >= 1024 queries) gives the
    oracle's leaves, and the same leaves as the thread-per-tree kernel."""
    import torch

    from paper_1509_06957_b200.search import _route_device

    X = gaussian(rng, 3000 + nq, d)
    Xd, Q = X[:3000], X[3000:].copy()
    Q[::9, ::4] = 0.0
    Q[1::7, 1::5] = np.float32(2e-42)
    index = mrpt.grow_trees(Xd, T, depth, seed=4)
    ref = dict(matrices=[(R.col_ptr, R.row_idx, R.values) for R in index.matrices],
               splits=index.splits, leaf_offsets=index.leaf_offsets,
               leaf_indices=index.leaf_indices, depth=depth)
    want = np.asarray(O.query_leaves(Q, ref))
    D = index.device_index()
    Qd = torch.from_numpy(Q).cuda()
    got = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("MRPT_ROUTE_H32", mode)
        got[mode] = _route_device(Qd, D).cpu().numpy()
    assert np.array_equal(got["1"], want)
    assert np.array_equal(got["0"], want)


@pytest.mark.parametrize("n,d,T,depth,gen", [
    (100_000, 64, 3, 10, "gauss"),       # big-path segments (> 8192) at the top levels
    (60_000, 16, 2, 9, "ints"),          # heavy ties through the big path
    (40_000, 8, 2, 6, "ones"),           # all keys equal in a big segment
    (20_000, 32, 4, 12, "gauss"),        # tiny leaves (~5 points)
    (100_000, 8, 2, 7, "ones"),          # top levels: one value, lists beyond shared memory
    (120_001, 4, 2, 8, "tail"),          # top levels: bucket range sampled from a constant prefix
    (150_000, 16, 2, 11, "ints"),        # top levels with heavy ties, then the per-segment kernels
    (70_000, 6, 3, 5, "gauss"),          # every level on the top path
])
def test_build_matches_oracle_large(rng, n, d, T, depth, gen):
    if gen == "gauss":
        X = gaussian(rng, n, d)
    elif gen == "ints":
        X = rng.integers(0, 3, size=(n, d)).astype(np.float32)
    elif gen == "tail":
        X = gaussian(rng, n, d)
        X[:70_000] = 0.25
    else:
        X = np.ones((n, d), dtype=np.float32)
    index = mrpt.grow_trees(X, T, depth, seed=17)
    for t in range(T):
        R, (s, o, i) = O.build_one_tree(X, depth, 1 / np.sqrt(d), 17, t)
        assert index.splits[t].tobytes() == s.tobytes(), t
        assert np.array_equal(index.leaf_offsets[t], o), t
        assert np.array_equal(index.leaf_indices[t], i), t


def test_batched_build_equals_single_tree_batches(rng):
    X = gaussian(rng, 5000, 20)
    a = mrpt.grow_trees(X, 7, 6, seed=4, batch_trees=7)
    b = mrpt.grow_trees(X, 7, 6, seed=4, batch_trees=2)
    assert a.splits.tobytes() == b.splits.tobytes()
    assert np.array_equal(a.leaf_indices, b.leaf_indices)


@pytest.mark.parametrize("size", [1, 3, 4096, 4097, 1 << 20, 5_000_011])
def test_fnv_matches_oracle(rng, size):
    buf = rng.integers(0, 256, size=size).astype(np.uint8)
    assert mrpt.fnv1a64(buf) == O.fnv1a64(buf.tobytes())


@pytest.mark.parametrize("offset", [1, 3, 8])
def test_fnv_unaligned_and_many_chunks(rng, offset):
    """Device buffers not 16-byte aligned (staged byte-wise) and a size with
    many chunks plus a ragged last one."""
    import torch

    from paper_1509_06957_b200.core import fnv1a64_device

    buf = rng.integers(0, 256, size=40_000_013 + offset).astype(np.uint8)
    t = torch.from_numpy(buf).cuda()[offset:]
    assert fnv1a64_device(t) == O.fnv1a64(buf[offset:].tobytes())


def test_fnv_golden_vectors():
    g = golden("fnv.npz")
    blob = g["blob"].tobytes()
    off = 0
    for ln, h in zip(g["lens"], g["hashes"]):
        assert mrpt.fnv1a64(blob[off:off + int(ln)]) == int(h)
        off += int(ln)


def test_scan_bit_identical(rng):
    from paper_1509_06957_b200 import _native

    X = gaussian(rng, 2000, 96)
    q = gaussian(rng, 1, 96)[0]
    cand = rng.choice(2000, size=700, replace=False).astype(np.int64)
    torch = _device.torch_mod()
    out = torch.empty(700, dtype=torch.float64, device="cuda")
    Xd, cd, qd = _device.h2d(X), _device.h2d(cand), _device.h2d(q)
    _native.call("mrpt_scan", _native.ptr(Xd), 2000, 96, 96, _native.ptr(cd), 700,
                 _native.ptr(qd), _native.ptr(out), _native.stream_ptr())
    assert _device.d2h(out).tobytes() == O.scan(X, cand, q).tobytes()


def test_exact_knn_in_set_matches_oracle(rng):
    X = gaussian(rng, 500, 13)
    q = gaussian(rng, 1, 13)[0]
    cand = rng.integers(0, 500, size=300)  # with duplicates
    for k in (1, 7, 100, 400):
        r = mrpt.exact_knn_in_set(q, k, cand, X)
        ids, dists, cnt = O.exact_knn(X, q, k, cand)
        assert r.indices.tolist() == ids.tolist()
        assert r.distances.tobytes() == dists.tobytes()
        assert r.candidate_count == cnt


def test_large_k_multipass(rng):
    X = gaussian(rng, 9000, 8)
    q = gaussian(rng, 1, 8)[0]
    r = mrpt.exact_knn_in_set(q, 7000, np.arange(9000), X)
    ids, dists, cnt = O.exact_knn(X, q, 7000, np.arange(9000))
    assert r.indices.tolist() == ids.tolist()
    assert r.distances.tobytes() == dists.tobytes()


@pytest.mark.parametrize("T,depth,n", [(300, 8, 50_000), (40, 12, 400_000)])
def test_vote_tiled_and_wide_counters(rng, T, depth, n):
    """u16 counters (T > 255) and the multi-tile id sweep (n > one tile)."""
    c = 3.0 * rng.standard_normal((50, 16))
    X = (c[rng.integers(0, 50, size=n + 64)] + rng.standard_normal((n + 64, 16))).astype(np.float32)
    Xd, Q = X[:n], X[n:]
    index = mrpt.grow_trees(Xd, T, depth, seed=2)
    ref = dict(matrices=[(R.col_ptr, R.row_idx, R.values) for R in index.matrices],
               splits=index.splits, leaf_offsets=index.leaf_offsets,
               leaf_indices=index.leaf_indices, depth=depth)
    for v in (1, 3, T // 2):
        ids, dists, counts = mrpt.approximate_knn_batch(Q, 10, index, v)
        rids, rd, rc = O.approximate_knn_batch(Xd, Q, 10, ref, v)
        assert np.array_equal(counts.astype(np.int64), rc)
        assert np.array_equal(ids, rids)
        assert dists.tobytes() == rd.tobytes()


def test_vote_hash_overflow_falls_back_to_tiles(rng):
    """iid data: each query's leaves cover more distinct points than the hash
    table holds, so every query takes the exact tiled sweep."""
    n, T, depth = 300_000, 60, 8
    X = gaussian(rng, n + 40, 8)
    Xd, Q = X[:n], X[n:]
    index = mrpt.grow_trees(Xd, T, depth, seed=9)
    ref = dict(matrices=[(R.col_ptr, R.row_idx, R.values) for R in index.matrices],
               splits=index.splits, leaf_offsets=index.leaf_offsets,
               leaf_indices=index.leaf_indices, depth=depth)
    for v in (1, 2):
        ids, dists, counts = mrpt.approximate_knn_batch(Q, 10, index, v)
        rids, rd, rc = O.approximate_knn_batch(Xd, Q, 10, ref, v)
        assert np.array_equal(counts.astype(np.int64), rc)
        assert np.array_equal(ids, rids)
        assert dists.tobytes() == rd.tobytes()


def test_unsorted_foreign_index_multi_tile_matches(rng):
    """A loaded index whose leaf slices are not ascending (and n larger than
    one counter tile) is audited, voted by the filtering sweep, and answers
    exactly like the ascending original."""
    n, T, depth = 260_000, 12, 7
    X = gaussian(rng, n + 30, 6)
    Xd, Q = X[:n], X[n:]
    a = mrpt.grow_trees(Xd, T, depth, seed=4)
    li = a.leaf_indices.copy()
    for t in range(T):
        o = a.leaf_offsets[t]
        for j in range(len(o) - 1):
            seg = li[t, o[j]:o[j + 1]]
            li[t, o[j]:o[j + 1]] = seg[rng.permutation(len(seg))]
    b = mrpt.MRPTIndex(dataset=mrpt.Dataset(Xd), n_trees=T, depth=depth, sparsity=a.sparsity,
                       seed=4, fixed_count=False, matrices=a.matrices, splits=a.splits,
                       leaf_offsets=a.leaf_offsets, leaf_indices=li,
                       dataset_checksum=a.dataset_checksum)
    assert not b.device_index().leaves_sorted
    for v in (1, 3):
        ra = mrpt.approximate_knn_batch(Q, 7, a, v)
        rb = mrpt.approximate_knn_batch(Q, 7, b, v)
        for x, y in zip(ra, rb):
            assert np.array_equal(x, y)


def _vote_lists(index, Q, v):
    """Raw K2+K3 output (candidate lists, counts) through the C ABI."""
    import torch

    from paper_1509_06957_b200 import _native
    from paper_1509_06957_b200.search import _route_device

    D = index.device_index()
    Qd = torch.from_numpy(np.ascontiguousarray(Q)).cuda()
    leaves = _route_device(Qd, D)
    cap = D.cap(v)
    cand = torch.full((Q.shape[0], cap), -7, dtype=torch.int32, device="cuda")
    counts = torch.empty(Q.shape[0], dtype=torch.int32, device="cuda")
    _native.call("mrpt_vote", _native.ptr(D.indices), _native.ptr(D.offsets), D.n, D.T, D.depth,
                 _native.ptr(leaves), Q.shape[0], int(v), int(D.leaves_sorted), int(D.max_count),
                 _native.ptr(D.vote_dir()), _native.ptr(cand), int(cap), _native.ptr(counts),
                 _native.stream_ptr())
    c = counts.cpu().numpy()
    lists = [row[:m] for row, m in zip(cand.cpu().numpy(), c)]
    return lists, c


@pytest.mark.parametrize("T,depth,n,votes", [(12, 7, 260_000, (2, 3)),      # fewer trees than warps, u8
                                             (300, 6, 200_000, (1, 2, 9)),  # ranged warps, 10-bit counters
                                             (1000, 9, 150_000, (3, 10)),   # ranged, 31-32 trees per warp
                                             (1100, 5, 140_000, (2, 40))])  # 32-tree groups, u16
def test_vote_multi_tile_matches_oracle(rng, monkeypatch, T, depth, n, votes):
    """Several id tiles (fewer trees than warps, ranged warps, 32-tree
    groups; u8 / 10-bit / u16 counters): the directory-driven vote gives the
    oracle's candidate counts, neighbour ids and distances."""
    X = gaussian(rng, n + 40, 5)
    Xd, Q = X[:n], X[n:]
    index = mrpt.grow_trees(Xd, T, depth, seed=6)
    D = index.device_index()
    assert D.vote_dir() is not None and D.vote_dir().numel() > 0
    ref = dict(matrices=[(R.col_ptr, R.row_idx, R.values) for R in index.matrices],
               splits=index.splits, leaf_offsets=index.leaf_offsets,
               leaf_indices=index.leaf_indices, depth=depth)
    monkeypatch.setenv("MRPT_VOTE_UNION", "0")
    for v in votes:
        got, gc = _vote_lists(index, Q, v)
        ids, dists, counts = mrpt.approximate_knn_batch(Q, 10, index, v)
        rids, rd, rc = O.approximate_knn_batch(Xd, Q, 10, ref, v)
        assert np.array_equal(gc.astype(np.int64), rc)
        assert np.array_equal(counts.astype(np.int64), rc)
        assert np.array_equal(ids, rids)
        assert dists.tobytes() == rd.tobytes()


@pytest.mark.parametrize("T,depth,n,shuffle", [(40, 6, 20_000, False), (1100, 5, 3_000, False),
                                               (600, 6, 30_000, True), (6, 10, 900_000, False)])
def test_vote_union_v1_matches_counting_path(rng, monkeypatch, T, depth, n, shuffle):
    """v = 1 runs the bitmap-union kernel (512 or 1024 threads, ranged or
    32-tree-group warps, sorted or shuffled slices); its candidate lists are
    identical, element for element, to the counting kernels' and the
    oracle's."""
    X = gaussian(rng, n + 24, 6)
    Xd, Q = X[:n], X[n:]
    index = mrpt.grow_trees(Xd, T, depth, seed=5)
    if shuffle:
        li = index.leaf_indices.copy()
        for t in range(T):
            o = index.leaf_offsets[t]
            for j in range(len(o) - 1):
                li[t, o[j]:o[j + 1]] = li[t, o[j]:o[j + 1]][rng.permutation(o[j + 1] - o[j])]
        index = mrpt.MRPTIndex(dataset=mrpt.Dataset(Xd), n_trees=T, depth=depth,
                               sparsity=index.sparsity, seed=5, fixed_count=False,
                               matrices=index.matrices, splits=index.splits,
                               leaf_offsets=index.leaf_offsets, leaf_indices=li,
                               dataset_checksum=index.dataset_checksum)
    monkeypatch.setenv("MRPT_VOTE_UNION", "1")
    got, gc = _vote_lists(index, Q, 1)
    monkeypatch.setenv("MRPT_VOTE_UNION", "0")
    want, wc = _vote_lists(index, Q, 1)
    assert np.array_equal(gc, wc)
    for a, b in zip(got, want):
        assert np.array_equal(a, np.sort(b))
        assert np.all(np.diff(a) > 0)
    monkeypatch.setenv("MRPT_VOTE_UNION", "1")
    ref = dict(matrices=[(R.col_ptr, R.row_idx, R.values) for R in index.matrices],
               splits=index.splits, leaf_offsets=index.leaf_offsets,
               leaf_indices=index.leaf_indices, depth=depth)
    ids, dists, counts = mrpt.approximate_knn_batch(Q, 10, index, 1)
    rids, rd, rc = O.approximate_knn_batch(Xd, Q, 10, ref, 1)
    assert np.array_equal(counts.astype(np.int64), rc)
    assert np.array_equal(ids, rids)
    assert dists.tobytes() == rd.tobytes()


def test_pipelined_host_batch_matches(rng):
    """Large host batches take the overlapped upload/compute/download path
    (numpy, pinned and pageable tensors); results equal the one-shot device
    path and the oracle."""
    import torch

    n, d = 20_000, 16
    X = gaussian(rng, n + 9000, d)
    Xd, Q = X[:n], X[n:]
    index = mrpt.grow_trees(Xd, 8, 6, seed=12)
    want = mrpt.approximate_knn_batch(Q, 6, index, 2, chunk=len(Q))  # unpipelined
    got_np = mrpt.approximate_knn_batch(Q, 6, index, 2)
    got_pin = mrpt.approximate_knn_batch(torch.from_numpy(Q).pin_memory(), 6, index, 2)
    got_page = mrpt.approximate_knn_batch(torch.from_numpy(Q.copy()), 6, index, 2)
    for got in (got_np, got_pin, got_page):
        for a, b in zip(got, want):
            assert isinstance(a, np.ndarray)
            assert np.array_equal(a, b)
    ref = dict(matrices=[(R.col_ptr, R.row_idx, R.values) for R in index.matrices],
               splits=index.splits, leaf_offsets=index.leaf_offsets,
               leaf_indices=index.leaf_indices, depth=6)
    rids, rd, rc = O.approximate_knn_batch(Xd, Q[:60], 6, ref, 2)
    assert np.array_equal(got_np[0][:60], rids)
    assert got_np[1][:60].tobytes() == rd.tobytes()
    assert np.array_equal(got_np[2][:60].astype(np.int64), rc)


@pytest.mark.parametrize("n,T,depth,votes", [(20_000, 12, 7, (1, 2, 4)),
                                             (300_000, 40, 9, (1, 3, 6)),
                                             (8_000, 300, 5, (2, 10, 40))])
def test_vote_sweep_one_pass_matches_per_threshold(rng, n, T, depth, votes):
    """approximate_knn_sweep (one route + one counted vote, filtered per
    threshold) answers every threshold exactly like approximate_knn_batch
    and like the oracle."""
    X = gaussian(rng, n + 40, 10)
    Xd, Q = X[:n], X[n:]
    index = mrpt.grow_trees(Xd, T, depth, seed=17)
    sweep = mrpt.approximate_knn_sweep(Q, 7, index, votes)
    assert sorted(sweep) == sorted(votes)
    ref = dict(matrices=[(R.col_ptr, R.row_idx, R.values) for R in index.matrices],
               splits=index.splits, leaf_offsets=index.leaf_offsets,
               leaf_indices=index.leaf_indices, depth=depth)
    for v in votes:
        ids, dists, counts = sweep[v]
        bids, bd, bc = mrpt.approximate_knn_batch(Q, 7, index, v)
        assert np.array_equal(ids, bids) and dists.tobytes() == bd.tobytes()
        assert np.array_equal(counts, bc)
        rids, rd, rc = O.approximate_knn_batch(Xd, Q, 7, ref, v)
        assert np.array_equal(ids, rids)
        assert dists.tobytes() == rd.tobytes()
        assert np.array_equal(counts.astype(np.int64), rc)


def test_vote_sweep_in_query_chunks(rng, monkeypatch):
    """A sweep whose scratch budget holds only 7 queries at a time gives the
    same answers as the one-chunk sweep (40 queries: five full chunks + 5)."""
    from paper_1509_06957_b200 import search

    X = gaussian(rng, 20_040, 10)
    Xd, Q = X[:20_000], X[20_000:]
    index = mrpt.grow_trees(Xd, 12, 7, seed=17)
    whole = mrpt.approximate_knn_sweep(Q, 7, index, (1, 2, 4))
    D = index.device_index()
    monkeypatch.setattr(search, "_SWEEP_SCRATCH_BYTES", 7 * (4 * D.T + 6 * D.cap(1)))
    parts = mrpt.approximate_knn_sweep(Q, 7, index, (1, 2, 4))
    for v in (1, 2, 4):
        for a, b in zip(whole[v], parts[v]):
            assert a.tobytes() == b.tobytes()


def _stream_lists(index, Q, v, cap=None, layout="stream"):
    """Raw K2 + streamed K3 output through the C ABI (mrpt_vote_stream, or
    mrpt_vote_pair over the paired layout)."""
    import torch

    from paper_1509_06957_b200 import _native
    from paper_1509_06957_b200.search import _route_device

    D = index.device_index()
    vs = D.vote_pair() if layout == "pair" else D.vote_stream()
    assert vs is not None, "the streamed layout should apply here"
    qs, tstride, qdir, qbase = vs
    Qd = torch.from_numpy(np.ascontiguousarray(Q)).cuda()
    leaves = _route_device(Qd, D)
    cap = D.cap(v) if cap is None else cap
    cand = torch.full((Q.shape[0], cap), -7, dtype=torch.int32, device="cuda")
    counts = torch.empty(Q.shape[0], dtype=torch.int32, device="cuda")
    _native.call("mrpt_vote_pair" if layout == "pair" else "mrpt_vote_stream", _native.ptr(qs),
                 int(tstride), _native.ptr(qdir), _native.ptr(qbase), D.n, D.T, D.depth, int(D.max_count),
                 _native.ptr(leaves), Q.shape[0], int(v), _native.ptr(cand), int(cap),
                 _native.ptr(counts), _native.stream_ptr())
    c = counts.cpu().numpy()
    return [row[:min(m, cap)] for row, m in zip(cand.cpu().numpy(), c)], c


@pytest.mark.parametrize("T,depth,n,kind,votes", [
    (12, 7, 500_000, "gauss", (1, 2, 12)),     # u8 counters, fewer trees than warps, 3 tiles
    (300, 6, 400_000, "ints", (2, 9, 300)),    # 10-bit counters, ties (unbalanced leaves)
    (1000, 9, 400_000, "gauss", (3, 10)),      # 31-32 trees per warp
    (1024, 5, 250_000, "gauss", (2, 40)),      # u16 counters (T = 1024 > 1023)
    (40, 4, 223_233, "gauss", (1, 5)),         # u8 counters: a last tile of one id
])
def test_streamed_vote_matches_oracle(rng, T, depth, n, kind, votes):
    """The streamed tiled vote (padded, pre-decoded leaf slices) gives the
    oracle's candidate sets and counts, and the batch API over it the
    oracle's neighbour ids and distances."""
    if kind == "ints":
        X = rng.integers(0, 40, size=(n + 40, 5)).astype(np.float32)
    else:
        X = gaussian(rng, n + 40, 5)
    Xd, Q = X[:n], X[n:]
    index = mrpt.grow_trees(Xd, T, depth, seed=8)
    ref = dict(matrices=[(R.col_ptr, R.row_idx, R.values) for R in index.matrices],
               splits=index.splits, leaf_offsets=index.leaf_offsets,
               leaf_indices=index.leaf_indices, depth=depth)
    leaves = O.query_leaves(Q, ref)
    pair_max = index.device_index().pair_max_votes()
    assert pair_max == (128 if T > 255 else T)  # T > 255 here: saturating u8 counters (fewer tile pairs)
    for v in votes:
        for layout in ("stream", "pair"):
            if layout == "pair" and v > pair_max:
                with pytest.raises(mrpt.ParameterError):
                    _stream_lists(index, Q, v, layout=layout)
                continue  # approximate_knn_batch below serves it with mrpt_vote
            got, gc = _stream_lists(index, Q, v, layout=layout)
            for i in range(len(Q)):
                want = O.candidates(leaves[i], ref, v)
                assert gc[i] == len(want)
                assert np.array_equal(np.sort(got[i]), want)
        ids, dists, counts = mrpt.approximate_knn_batch(Q, 10, index, v)
        rids, rd, rc = O.approximate_knn_batch(Xd, Q, 10, ref, v)
        assert np.array_equal(counts.astype(np.int64), rc)
        assert np.array_equal(ids, rids)
        assert dists.tobytes() == rd.tobytes()


@pytest.mark.parametrize("T,depth,n,dim,votes", [
    (1000, 9, 400_000, 5, (3, 10, 128)),   # counts far above 255: every hot id is pulled back several times
    (300, 5, 350_000, 5, (1, 7)),          # 2 tiles of 8-bit counters (3 of 10-bit ones), big leaves
])
def test_saturating_pair_vote_and_its_exact_redo(rng, monkeypatch, T, depth, n, dim, votes):
    """T > 255 with 8-bit counters: the saturating paired vote lists exactly
    the oracle's candidates (counts reach hundreds, so the pull-back runs all
    the time), and so does the check-before-increment redo that a wrapped
    counter would trigger (forced here for every query by MRPT_VOTE_DBG=8)."""
    from paper_1509_06957_b200.search import vote_stats

    X = gaussian(rng, n + 24, dim)
    Xd, Q = X[:n], np.concatenate([X[n:], X[:8]])  # 8 queries are data points
    index = mrpt.grow_trees(Xd, T, depth, seed=5)
    ref = dict(matrices=[(R.col_ptr, R.row_idx, R.values) for R in index.matrices],
               splits=index.splits, leaf_offsets=index.leaf_offsets,
               leaf_indices=index.leaf_indices, depth=depth)
    leaves = O.query_leaves(Q, ref)
    want = {v: [O.candidates(leaves[i], ref, v) for i in range(len(Q))] for v in votes}
    top = max(int(np.bincount(np.concatenate([index.leaf_indices[t, index.leaf_offsets[t, f]:index.leaf_offsets[t, f + 1]]
                                              for t, f in enumerate(leaves[-1])])).max()), 0)
    assert top > 255, "the case should count past 8 bits"
    for forced in (False, True):
        if forced:
            monkeypatch.setenv("MRPT_VOTE_DBG", "8")
        vote_stats(reset=True)
        for v in votes:
            got, gc = _stream_lists(index, Q, v, layout="pair")
            for i in range(len(Q)):
                assert gc[i] == len(want[v][i])
                assert np.array_equal(np.sort(got[i]), want[v][i])
        st = vote_stats()
        assert st["queries"] == len(votes) * len(Q)
        print(f"T={T} forced={forced}: saturating vote {st}")
        if forced:
            assert st["redone"] == len(votes) * len(Q)


def test_streamed_vote_layout_round_trip(rng):
    """Decoding the streamed layout (quads -> ids, padding dropped) gives back
    every leaf slice exactly: the layout is a lossless re-encoding."""
    T, depth, n = 7, 6, 300_000
    X = gaussian(rng, n, 4)
    index = mrpt.grow_trees(X, T, depth, seed=2)
    D = index.device_index()
    qs, tstride, qdir, qbase = D.vote_stream()
    qs = qs.cpu().numpy().view(np.uint32).reshape(T, tstride, 4)
    qbase = qbase.cpu().numpy()
    L = 1 << depth
    nt = qdir.numel() // (T * L) - 1
    qdir = qdir.cpu().numpy().view(np.uint16).reshape(T, L, nt + 1).astype(np.int64)
    words = ((218 * 1024 - 128) // 4) & ~3
    W = words * 4  # u8 counters (T <= 255): 4 ids per counter word
    pad_word = (W // 4 + 3) & ~3  # padding entries address spare words from here on
    assert nt == -(-n // W)
    offs, li = index.leaf_offsets, index.leaf_indices
    for t in range(T):
        for f in range(L):
            s0 = qbase[t * L + f]
            ids = []
            for w in range(nt):
                # a quad: u16 counter words of 7 entries, then their 2-bit lanes
                quads = qs[t, s0 + qdir[t, f, w]: s0 + qdir[t, f, w + 1]].view(np.uint16)
                for u in quads.reshape(-1, 8):
                    fb = int(u[7])
                    for i in range(7):
                        if u[i] < pad_word:
                            ids.append(w * W + int(u[i]) * 4 + ((fb >> (2 * i)) & 3))
                        else:
                            assert u[i] < pad_word + 32 and (fb >> (2 * i)) & 3 == 0
            assert np.array_equal(np.array(ids, dtype=np.int64), li[t, offs[t, f]:offs[t, f + 1]])


def test_paired_vote_layout_round_trip(rng):
    """Decoding the paired layout (pairs -> the two tiles' quads -> ids,
    padding dropped) gives back every leaf slice exactly, with an odd tile
    count (the last super-tile's second quads are all padding)."""
    T, depth, n = 5, 6, 2 * 223_104 + 17  # u8 counters: 223,104 ids per tile -> 3 tiles
    X = gaussian(rng, n, 4)
    index = mrpt.grow_trees(X, T, depth, seed=3)
    D = index.device_index()
    ps, pstride, pdir, pbase = D.vote_pair()
    ps = ps.cpu().numpy().view(np.uint32).reshape(T, pstride, 2, 4)
    pbase = pbase.cpu().numpy()
    L = 1 << depth
    words = ((218 * 1024 - 128) // 4) & ~3
    W = words * 4
    nt = -(-n // W)
    nsup = (nt + 1) // 2
    assert pdir.numel() == T * L * (nsup + 1)
    pdir = pdir.cpu().numpy().view(np.uint16).reshape(T, L, nsup + 1).astype(np.int64)
    pad_word = (W // 4 + 3) & ~3
    offs, li = index.leaf_offsets, index.leaf_indices
    for t in range(T):
        for f in range(L):
            s0 = pbase[t * L + f]
            ids = []
            for j in range(nsup):
                pairs = ps[t, s0 + pdir[t, f, j]: s0 + pdir[t, f, j + 1]]
                for side in (0, 1):
                    w = 2 * j + side
                    for u in pairs[:, side].copy().view(np.uint16).reshape(-1, 8):
                        fb = int(u[7])
                        for i in range(7):
                            if u[i] < pad_word:
                                assert w < nt
                                ids.append(w * W + int(u[i]) * 4 + ((fb >> (2 * i)) & 3))
                            else:
                                assert u[i] < pad_word + 32 and (fb >> (2 * i)) & 3 == 0
            assert np.array_equal(np.sort(np.array(ids, dtype=np.int64)), li[t, offs[t, f]:offs[t, f + 1]])
