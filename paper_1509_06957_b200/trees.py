"""Random projection tree construction on the GPU (mirrors pkg/src/mrpt/trees.py).

``grow_trees`` keeps the reference's signature, validation and results:
tree t uses the matrix drawn from (seed, t) (host numpy, bit-exact), the
projections are computed by K1 (``mrpt_project``) into a level-major
(Tb, depth, n) buffer, and K5 (``mrpt_build_levels``) splits every node of
every tree in the batch level by level at the exact lower median with a
stable partition -- the same splits, leaf offsets and leaf id order the
reference produces (trees.py:54-98, 187-245).  The index stays on the
device; the host arrays the reference exposes are materialised on demand.
"""

from __future__ import annotations

import ctypes
import math
import os
import threading

import numpy as np

from . import _device, _native
from .core import (
    Dataset,
    SparseProjectionMatrix,
    _record_macs,
    as_dataset,
    default_sparsity,
    sample_sparse_matrix,
)
from .exceptions import DepthError, IntegrityError, MRPTError, ParameterError

__all__ = ["MRPTIndex", "RPTree", "build_tree", "grow_trees", "median_split"]


def _as_f32_values(values):
    """float32 copy of ``values``; the GPU compares in float32, so inputs whose
    values float32 cannot hold exactly are rejected rather than silently
    re-rounded."""
    v = np.asarray(values)
    f = np.ascontiguousarray(v, dtype=np.float32)
    if v.dtype != np.float32:
        with np.errstate(invalid="ignore", over="ignore"):
            if not np.array_equal(f.astype(v.dtype), v, equal_nan=True):
                raise ParameterError("projection values must be exactly representable in float32 "
                                     "(the device split kernels compare in float32)")
    return f


def _build_device(Pdev, n, Tb, depth, splits, offsets, indices):
    """Run K5 on a (Tb, depth, n) projection buffer into the given outputs."""
    torch = _device.torch_mod()
    sz = ctypes.c_size_t(0)
    _native.call("mrpt_build_workspace_size", n, Tb, depth, ctypes.byref(sz))
    ws = torch.empty(max(1, sz.value), dtype=torch.uint8, device=Pdev.device)
    _native.call("mrpt_build_levels", _native.ptr(Pdev), n, Tb, depth, _native.ptr(splits),
                 _native.ptr(offsets), _native.ptr(indices), _native.ptr(ws), sz.value,
                 _native.stream_ptr())


def _single_tree(P_rows_f32, depth):
    """Build one tree over an (n, depth) host float32 matrix on the GPU."""
    torch = _device.torch_mod()
    n = P_rows_f32.shape[0]
    Pd = _device.h2d(np.ascontiguousarray(P_rows_f32[:, :depth].T))  # level-major
    splits = torch.empty((1, (1 << depth) - 1), dtype=torch.float32, device=Pd.device)
    offsets = torch.empty((1, (1 << depth) + 1), dtype=torch.int64, device=Pd.device)
    order = torch.empty((1, n), dtype=torch.int32, device=Pd.device)
    _build_device(Pd, n, 1, depth, splits, offsets, order)
    return _device.d2h(splits)[0], _device.d2h(offsets)[0], _device.d2h(order)[0]


def median_split(values, indices):
    """Split ``indices`` at the lower median of ``values`` (trees.py:33-51).

    split = the ceil(m/2)-th smallest value; entries with value <= split go
    left in their original order, the rest right.  Runs as a one-level build
    on the device.
    """
    v = np.asarray(values)
    idx = np.asarray(indices)
    m = v.shape[0]
    if m < 2:
        raise ParameterError(f"median_split needs at least 2 entries, got {m}")
    f = _as_f32_values(v)
    splits, offsets, order = _single_tree(f.reshape(m, 1), 1)
    nle = int(offsets[1])
    split = v.dtype.type(splits[0]) if np.issubdtype(v.dtype, np.floating) else splits[0]
    return split, idx[order[:nle]], idx[order[nle:]]


def build_tree(P, depth, indices=None):
    """Grow one tree from precomputed projections ``P`` (n x depth), trees.py:54-98.

    Returns (splits f32[2^depth-1], leaf_offsets i64[2^depth+1], order i32).
    With ``indices`` the tree is built over those rows of P in that order.
    """
    P = np.asarray(P)
    if depth < 0 or P.ndim != 2 or P.shape[1] < depth:
        raise ParameterError(f"projection matrix has {P.shape[1] if P.ndim == 2 else 0} levels, "
                             f"need {depth}")
    order0 = (np.arange(P.shape[0], dtype=np.int32) if indices is None
              else np.array(indices, dtype=np.int32))
    nleaf = 1 << depth
    if depth == 0 or order0.shape[0] == 0:
        splits = np.zeros(nleaf - 1, dtype=np.float32)
        bounds = np.zeros(nleaf + 1, dtype=np.int64)
        bounds[1:] = order0.shape[0]
        if depth > 0:
            bounds[:] = 0
        return splits, bounds, order0
    rows = P if indices is None else P[order0]
    splits, offsets, pos = _single_tree(_as_f32_values(rows), depth)
    order = pos if indices is None else order0[pos]
    return splits, offsets, np.ascontiguousarray(order, dtype=np.int32)


from dataclasses import dataclass  # noqa: E402


@dataclass(frozen=True)
class RPTree:
    """One tree of an index: its matrix plus the flat tree arrays (trees.py:101-121)."""

    random_matrix: SparseProjectionMatrix
    depth: int
    splits: np.ndarray  # float32 (2^depth - 1,)
    leaf_offsets: np.ndarray  # int64 (2^depth + 1,)
    leaf_indices: np.ndarray  # int32 (n,)

    @property
    def n_leaves(self):
        return 2 ** self.depth

    def leaf(self, leaf_id):
        s, e = self.leaf_offsets[leaf_id], self.leaf_offsets[leaf_id + 1]
        return self.leaf_indices[s:e].copy()

    def leaf_sizes(self):
        return np.diff(self.leaf_offsets)


class _DeviceIndex:
    """Device-resident copy of an index, as the query kernels consume it."""

    def __init__(self, X, T, depth, splits, offsets, indices, col_ptr, rows, vals, leaves_sorted,
                 max_count, max_leaf):
        self.X = X
        self.n, self.d = int(X.shape[0]), int(X.shape[1])
        self.T, self.depth = T, depth
        self.splits, self.offsets, self.indices = splits, offsets, indices
        self.col_ptr, self.rows, self.vals = col_ptr, rows, vals
        self.leaves_sorted = leaves_sorted
        self.max_count = max_count
        self.max_leaf = max_leaf
        self.scan_choice = {}  # (k, votes) -> exact route chosen by the autotune
        self.scan_choice_by_size = {}  # (k, votes, batch-size class) -> route
        self.scan_pin = {}  # (k, votes) -> route forced for every batch size (pin_route)
        self._ws = {}  # (name, stream) -> scratch
        self._ws_lock = threading.Lock()

    def cap(self, votes):
        """Upper bound on any candidate set at this vote threshold."""
        return max(1, min(self.n, (self.T * self.max_leaf) // votes))

    def shadow(self):
        """(fp16 rows, row stride, radius) for the scan filter, built once; None
        when not worth it, or the rows do not fit the kernel or the fp16 range."""
        if getattr(self, "_shadow", False) is not False:
            return self._shadow
        self._shadow = None
        ldh = (self.d + 7) // 8 * 8
        # worth it when the candidate rows stream from HBM (X well beyond L2)
        # and a row fills whole warps; MRPT_FP16_FILTER=1/0 forces it on/off
        mode = os.environ.get("MRPT_FP16_FILTER", "auto")
        if os.environ.get("MRPT_SCAN_ROWS") == "fp16":
            mode = "1"
        elif os.environ.get("MRPT_SCAN_ROWS") == "fp32":
            mode = "0"
        want = (mode == "1") or (mode == "auto" and self.d >= 256 and self.n * self.d * 4 > (256 << 20))
        if want and ldh <= 1024 and self.d % 4 == 0:
            torch = _device.torch_mod()
            Xh = torch.empty((self.n, ldh), dtype=torch.float16, device=self.X.device)
            rad = torch.empty(self.n, dtype=torch.float32, device=self.X.device)
            bad = torch.zeros(1, dtype=torch.int32, device=self.X.device)
            _native.call("mrpt_quantize_fp16", _native.ptr(self.X), self.n, self.d,
                         int(self.X.stride(0)), _native.ptr(Xh), ldh, _native.ptr(rad),
                         _native.ptr(bad), _native.stream_ptr())
            if not int(bad.item()):
                self._shadow = (Xh, ldh, rad)
        return self._shadow

    def u8_rows(self):
        """u8 shadow (rows, row stride, scale, norm, radius) for non-negative
        data, built once; None for signed data or unsupported widths
        (MRPT_SCAN_ROWS=fp16|fp32 disables it)."""
        if getattr(self, "_u8", False) is not False:
            return self._u8
        self._u8 = None
        ldq = (self.d + 15) // 16 * 16
        mode = os.environ.get("MRPT_SCAN_ROWS", "auto")
        if mode in ("auto", "u8", "u8tc_bits") and ldq <= 1024:
            torch = _device.torch_mod()
            dev = self.X.device
            Xq = torch.empty((self.n, ldq), dtype=torch.uint8, device=dev)
            sc = torch.empty(self.n, dtype=torch.float32, device=dev)
            nm = torch.empty(self.n, dtype=torch.int32, device=dev)
            rad = torch.empty(self.n, dtype=torch.float32, device=dev)
            flags = torch.zeros(2, dtype=torch.int32, device=dev)
            _native.call("mrpt_quantize_u8", _native.ptr(self.X), self.n, self.d,
                         int(self.X.stride(0)), _native.ptr(Xq), ldq, _native.ptr(sc),
                         _native.ptr(nm), _native.ptr(rad), _native.ptr(flags),
                         _native.stream_ptr())
            if not int(flags[0].item()):
                self._u8 = (Xq, ldq, sc, nm, rad)
        return self._u8

    def tc_rows(self):
        """(s8 rows, per-row records) of the fused tcgen05 filter over the u8
        shadow (mrpt_u8_gemm_rows), built once; None without a u8 shadow."""
        u8 = self.u8_rows()
        if u8 is None:
            return None
        if getattr(self, "_tcr", None) is None:
            torch = _device.torch_mod()
            Xq, ldq = u8[0], u8[1]
            Xs = torch.empty(((self.n + 15) // 16 * 16, ldq), dtype=torch.uint8, device=Xq.device)
            info = torch.empty((self.n, 4), dtype=torch.int32, device=Xq.device)
            _native.call("mrpt_u8_gemm_rows", _native.ptr(Xq), self.n, ldq, _native.ptr(u8[2]),
                         _native.ptr(u8[3]), _native.ptr(u8[4]), _native.ptr(Xs),
                         _native.ptr(info), _native.stream_ptr())
            self._tcr = (Xs, info)
        return self._tcr

    def workspace(self, name, nbytes):
        """A device scratch buffer of at least ``nbytes`` for this index, one per
        (name, caller stream): calls on different streams never share scratch
        (the reference's kernels are reentrant; so are these calls)."""
        torch = _device.torch_mod()
        key = (name, torch.cuda.current_stream().cuda_stream)
        with self._ws_lock:
            ws = self._ws.get(key)
            if ws is None or ws.numel() < nbytes:
                ws = self._ws[key] = torch.empty(max(1, int(nbytes)), dtype=torch.uint8,
                                                 device=self.X.device)
            return ws

    def pin_route(self, k, votes, route):
        """Force the exact K4 route for (k, votes) at every batch size (tools,
        tests); None unpins (the autotune decides again)."""
        if route is None:
            self.scan_pin.pop((k, votes), None)
        else:
            self.scan_pin[(k, votes)] = route
            self.scan_choice[(k, votes)] = route

    def u8_tc(self, nq):
        """(s8 rows, per-row records, workspace) for the fused tcgen05 filter
        (mrpt_scan_topk_u8tc_bits): rows built once, the workspace sized for
        nq queries and private to the caller's stream."""
        g = self.tc_rows()
        if g is None:
            return None
        need = ctypes.c_int64(0)
        _native.call("mrpt_scan_topk_u8tc_workspace_size", self.n, self.u8_rows()[1], int(nq),
                     ctypes.byref(need))
        return g[0], g[1], self.workspace("u8tc", need.value)

    def vote_stream(self):
        """The streamed-vote layout of this index (mrpt_vote_stream_layout /
        _fill: every leaf slice's per-id-tile pieces padded to 16-byte quads of
        pre-decoded counter addresses), built once on the device; None where
        one id tile covers the index, the slices are not ascending (foreign
        index), T > 1024, or it does not fit beside the index
        (MRPT_VOTE_STREAM=0 disables it)."""
        if getattr(self, "_vstream", False) is not False:
            return self._vstream
        self._vstream = None
        if os.environ.get("MRPT_VOTE_STREAM", "1") == "0":
            return None
        if not self.leaves_sorted or self.max_leaf > 65535 or self.T > 1024:
            return None
        ntiles, entries = ctypes.c_int32(0), ctypes.c_int64(0)
        try:
            _native.call("mrpt_vote_stream_plan", self.n, self.T, self.depth, int(self.max_count),
                         ctypes.byref(ntiles), ctypes.byref(entries))
        except MRPTError:
            return None
        nleaf = 1 << self.depth
        # padded lengths (7 ids per quad) must fit the u16 quad directory
        if ntiles.value <= 1 or (self.max_leaf + 6 * ntiles.value) // 7 >= 65535:
            return None
        torch = _device.torch_mod()
        dev = self.indices.device
        qdir = torch.empty(entries.value, dtype=torch.int16, device=dev)
        qbase = torch.empty(self.T * nleaf, dtype=torch.int32, device=dev)
        tq = torch.empty(self.T, dtype=torch.int64, device=dev)
        _native.call("mrpt_vote_stream_layout", _native.ptr(self.indices), _native.ptr(self.offsets),
                     self.n, self.T, self.depth, int(self.max_count), _native.ptr(qdir),
                     _native.ptr(qbase), _native.ptr(tq), _native.stream_ptr())
        tstride = int(tq.max().item())
        tstride = (tstride + 1) // 2 * 2  # 32-byte aligned tree rows
        nbytes = 16 * self.T * tstride
        free = torch.cuda.mem_get_info(dev)[0]
        if 32 * tstride >= (1 << 31) or nbytes > 0.8 * free:
            return None
        qs = torch.empty(nbytes // 4, dtype=torch.int32, device=dev)
        _native.call("mrpt_vote_stream_fill", _native.ptr(self.indices), _native.ptr(self.offsets),
                     self.n, self.T, self.depth, int(self.max_count), _native.ptr(qdir),
                     _native.ptr(qbase), tstride, _native.ptr(qs), _native.stream_ptr())
        self._vstream = (qs, tstride, qdir, qbase)
        return self._vstream

    def vote_pair(self):
        """The paired streamed-vote layout of this index (mrpt_vote_pair_layout
        / _fill: id tiles taken two at a time, every leaf slice stored as
        32-byte pairs of pre-decoded quads, one of each tile), built once on
        the device; None where the streamed layout would be None, or
        MRPT_VOTE_PAIR=0."""
        if getattr(self, "_vpair", False) is not False:
            return self._vpair
        self._vpair = None
        if os.environ.get("MRPT_VOTE_STREAM", "1") == "0" or os.environ.get("MRPT_VOTE_PAIR", "1") == "0":
            return None
        if not self.leaves_sorted or self.max_leaf > 65535 or self.T > 1024:
            return None
        ntiles, pos_n, dir_n = ctypes.c_int32(0), ctypes.c_int64(0), ctypes.c_int64(0)
        try:
            _native.call("mrpt_vote_pair_plan", self.n, self.T, self.depth, int(self.max_count),
                         ctypes.byref(ntiles), ctypes.byref(pos_n), ctypes.byref(dir_n))
        except MRPTError:
            return None
        nleaf = 1 << self.depth
        # padded lengths (7 ids per quad) must fit the u16 pair directory
        if ntiles.value <= 1 or (self.max_leaf + 6 * ntiles.value) // 7 >= 65535:
            return None
        torch = _device.torch_mod()
        dev = self.indices.device
        pos = torch.empty(pos_n.value, dtype=torch.int16, device=dev)
        pdir = torch.empty(dir_n.value, dtype=torch.int16, device=dev)
        pbase = torch.empty(self.T * nleaf, dtype=torch.int32, device=dev)
        tp = torch.empty(self.T, dtype=torch.int64, device=dev)
        _native.call("mrpt_vote_pair_layout", _native.ptr(self.indices), _native.ptr(self.offsets),
                     self.n, self.T, self.depth, int(self.max_count), _native.ptr(pos), _native.ptr(pdir),
                     _native.ptr(pbase), _native.ptr(tp), _native.stream_ptr())
        pstride = int(tp.max().item())
        nbytes = 32 * self.T * pstride
        free = torch.cuda.mem_get_info(dev)[0]
        if 64 * pstride >= (1 << 31) or nbytes > 0.8 * free:
            return None
        ps = torch.empty(nbytes // 4, dtype=torch.int32, device=dev)
        _native.call("mrpt_vote_pair_fill", _native.ptr(self.indices), _native.ptr(self.offsets),
                     self.n, self.T, self.depth, int(self.max_count), _native.ptr(pos), _native.ptr(pdir),
                     _native.ptr(pbase), pstride, _native.ptr(ps), _native.stream_ptr())
        del pos  # stream-ordered: the allocator reuses it only after the fill
        self._vpair = (ps, pstride, pdir, pbase)
        return self._vpair

    def pair_max_votes(self):
        """Largest vote threshold mrpt_vote_pair serves on this index (128
        where it votes with saturating 8-bit counters: T > 255 and large n)."""
        mv = ctypes.c_int32(0)
        _native.call("mrpt_vote_pair_max_votes", self.n, self.T, int(self.max_count), ctypes.byref(mv))
        return mv.value

    def vote_layout(self):
        """Which list-vote layout queries use: "pair" (mrpt_vote_pair),
        "stream" (mrpt_vote_stream) or None (mrpt_vote over leaf_indices)."""
        if self.vote_pair() is not None:
            return "pair"
        if self.vote_stream() is not None:
            return "stream"
        return None

    def vote_dir(self):
        """Tile directory for the multi-tile vote (built once, on the device),
        or None when one id tile covers the index or it cannot be used."""
        if getattr(self, "_dir", False) is not False:
            return self._dir
        self._dir = None
        if self.leaves_sorted and self.max_leaf <= 65535:
            ntiles, entries = ctypes.c_int32(0), ctypes.c_int64(0)
            _native.call("mrpt_vote_plan", self.n, self.T, self.depth, int(self.max_count),
                         ctypes.byref(ntiles), ctypes.byref(entries))
            if ntiles.value > 1:
                torch = _device.torch_mod()
                d = torch.empty(entries.value, dtype=torch.int16, device=self.indices.device)
                _native.call("mrpt_vote_build_dir", _native.ptr(self.indices),
                             _native.ptr(self.offsets), self.n, self.T, self.depth,
                             int(self.max_count), _native.ptr(d), _native.stream_ptr())
                self._dir = d
        return self._dir


class MRPTIndex:
    """T random projection trees over one dataset (trees.py:124-175).

    Same constructor fields as the reference dataclass, so hand-assembled or
    loaded indexes work; ``splits`` / ``leaf_offsets`` / ``leaf_indices`` may be
    host arrays or CUDA tensors.  Host views are materialised lazily for
    device-built indexes; the device copy is uploaded (and audited) lazily
    for host-built ones.
    """

    def __init__(self, dataset, n_trees, depth, sparsity, seed, fixed_count, matrices, splits,
                 leaf_offsets, leaf_indices, dataset_checksum, _local=None, _device_index=None):
        self.dataset = dataset
        self.n_trees = n_trees
        self.depth = depth
        self.sparsity = sparsity
        self.seed = seed
        self.fixed_count = fixed_count
        self.matrices = matrices
        self._arrays = {"splits": splits, "leaf_offsets": leaf_offsets,
                        "leaf_indices": leaf_indices}
        self.dataset_checksum = dataset_checksum
        self._local = _local if _local is not None else threading.local()
        self._dev = _device_index
        self._dev_lock = threading.Lock()

    def _host(self, name):
        a = self._arrays[name]
        if _device.is_tensor(a):
            a = _device.d2h(a)
            self._arrays[name] = a
        return a

    splits = property(lambda self: self._host("splits"),
                      lambda self, v: self._set("splits", v))
    leaf_offsets = property(lambda self: self._host("leaf_offsets"),
                            lambda self, v: self._set("leaf_offsets", v))
    leaf_indices = property(lambda self: self._host("leaf_indices"),
                            lambda self, v: self._set("leaf_indices", v))

    def _set(self, name, value):
        self._arrays[name] = value
        self._dev = None  # re-upload on next query

    def tree(self, t):
        return RPTree(random_matrix=self.matrices[t], depth=self.depth, splits=self.splits[t],
                      leaf_offsets=self.leaf_offsets[t], leaf_indices=self.leaf_indices[t])

    def __iter__(self):
        return (self.tree(t) for t in range(self.n_trees))

    @property
    def n(self):
        return self.dataset.n

    @property
    def d(self):
        return self.dataset.d

    def max_candidates(self):
        """T * ceil(n / 2^depth), the reference's bound (trees.py:161-163)."""
        return self.n_trees * math.ceil(self.n / 2 ** self.depth)

    def memory_bytes(self):
        nleaf = 1 << self.depth
        total = (self.n_trees * (nleaf - 1) * 4 + self.n_trees * (nleaf + 1) * 8
                 + self.n_trees * self.n * 4)
        for R in self.matrices:
            total += R.col_ptr.nbytes + R.row_idx.nbytes + R.values.nbytes
        return total

    def query(self, q, k, votes):
        from .search import approximate_knn

        return approximate_knn(q, k, self, votes)

    def __repr__(self):
        return (f"MRPTIndex(n={self.n}, d={self.d}, n_trees={self.n_trees}, depth={self.depth}, "
                f"sparsity={self.sparsity}, seed={self.seed})")

    # -- device side ---------------------------------------------------------
    def device_index(self):
        """The cached device copy (uploading and auditing it on first use)."""
        if self._dev is not None:
            return self._dev
        with self._dev_lock:
            if self._dev is None:
                self._dev = self._upload()
        return self._dev

    def _upload(self):
        torch = _device.torch_mod()
        T, depth, n = self.n_trees, self.depth, self.n
        nleaf = 1 << depth

        def dev(name, dtype, shape):
            a = self._arrays[name]
            if _device.is_tensor(a):
                t = a.to(device=_device.device(), dtype=dtype).contiguous()
            else:
                t = _device.h2d(np.asarray(a, dtype=np.dtype(str(dtype).split(".")[-1])))
            return t.reshape(shape)

        splits = dev("splits", torch.float32, (T, nleaf - 1))
        offsets = dev("leaf_offsets", torch.int64, (T, nleaf + 1))
        indices = dev("leaf_indices", torch.int32, (T, n))
        host_off = self._host("leaf_offsets").reshape(T, nleaf + 1)
        if (host_off[:, 0] != 0).any() or (host_off[:, -1] != n).any() or \
                (np.diff(host_off, axis=1) < 0).any():
            raise IntegrityError("leaf offsets must run from 0 to n without decreasing")
        flags = torch.zeros(2, dtype=torch.int32, device=indices.device)
        _native.call("mrpt_audit_leaves", _native.ptr(indices), _native.ptr(offsets), n, T, depth,
                     _native.ptr(flags), _native.stream_ptr())
        unsorted, out_of_range = (int(x) for x in _device.d2h(flags))
        if out_of_range:
            raise IntegrityError(f"leaf point ids must lie in [0, {n})")
        max_leaf = int(np.diff(host_off, axis=1).max())
        cp, rows, vals = _device.csc_device(self.matrices)
        return _DeviceIndex(self.dataset.device(), T, depth, splits, offsets, indices, cp, rows,
                            vals, leaves_sorted=not unsorted,
                            max_count=T if not unsorted else T * max(1, max_leaf),
                            max_leaf=max_leaf)


def _resolve_threads(threads):
    if threads is None:
        env = os.environ.get("MRPT_THREADS", "").strip()
        threads = int(env) if env else 1
    if threads < 1:
        raise ParameterError(f"thread count must be >= 1, got {threads}")
    return threads


def _batch_trees(n, d, depth, T, free_bytes):
    """Trees per K1+K5 batch: projections (depth*n*4) + keys + scratch order
    (8n) + top-level scratch per tree, within half of the free memory."""
    # + the top levels' node ids (2n) and per-run node tables (<= n/2) and fixed tables
    per_tree = n * (4 * depth + 8) + 3 * n + (1 << 20)
    tb = max(1, int(0.5 * free_bytes) // per_tree)
    tb = min(tb, T, 128)
    while tb > 1 and tb * (1 << depth) >= (1 << 31):
        tb //= 2
    # equal batches: the same number of launches without a small last batch
    # (config 5: 10 x 100 trees instead of 9 x 111 + 1; 1.77 vs 1.84 s)
    nb = -(-T // tb)
    return -(-T // nb)


def _validate_grow(X, n_trees, depth, sparsity, seed, threads):
    X = as_dataset(X)
    if n_trees < 1:
        raise ParameterError(f"tree count must be >= 1, got {n_trees}")
    if depth < 1:
        raise DepthError(f"depth must be >= 1, got {depth}")
    if 2 ** depth > X.n:
        raise DepthError(f"depth {depth} gives {2 ** depth} leaves but the dataset has only "
                         f"{X.n} points")
    if sparsity is None:
        sparsity = default_sparsity(X.d)
    seed = int(seed)
    if not 0 <= seed < 2 ** 64:
        raise ParameterError(f"seed must be an unsigned 64-bit integer, got {seed}")
    _resolve_threads(threads)
    if not 0.0 < sparsity <= 1.0:
        raise ParameterError(f"sparsity must lie in (0, 1], got {sparsity}")
    return X, float(sparsity), seed


def _grow_block(X, t_begin, t_end, depth, sparsity, seed, fixed_count, splits, offsets, indices,
                batch_trees=None, after_batch=None):
    """Build trees [t_begin, t_end) of an index (tree t from seed (seed, t)) into
    the device arrays ``splits/offsets/indices`` (rows 0 .. t_end-t_begin-1).
    Returns the host matrices of those trees.  No host synchronisation.
    ``after_batch(j)`` is called once the kernels of batch j are enqueued."""
    torch = _device.torch_mod()
    Xd = X.device()
    n, d = X.n, X.d
    dev = Xd.device
    count = t_end - t_begin
    free = torch.cuda.mem_get_info(dev)[0]
    tb = min(count, batch_trees or _batch_trees(n, d, depth, count, free))
    sz = ctypes.c_size_t(0)
    _native.call("mrpt_build_workspace_size", n, tb, depth, ctypes.byref(sz))
    ws = torch.empty(max(1, sz.value), dtype=torch.uint8, device=dev)
    P = torch.empty((tb, depth, n), dtype=torch.float32, device=dev)
    matrices = []
    stream = _native.stream_ptr()
    for b0 in range(0, count, tb):
        b1 = min(count, b0 + tb)
        mats = [sample_sparse_matrix(d, depth, sparsity, seed=(seed, t_begin + t),
                                     fixed_count=fixed_count) for t in range(b0, b1)]
        matrices.extend(mats)
        for R in mats:
            _record_macs(n * R.nnz)
        cp, rows, vals = _device.csc_device(mats, pinned=True)
        # K1: P[(t*depth + lev)*n + i] (row stride 1, column stride n)
        _native.call("mrpt_project", _native.ptr(Xd), n, d, d, _native.ptr(cp), _native.ptr(rows),
                     _native.ptr(vals), (b1 - b0) * depth, _native.ptr(P), 1, n, stream)
        # K5: all levels of the batch
        _native.call("mrpt_build_levels", _native.ptr(P), n, b1 - b0, depth,
                     _native.ptr(splits[b0:]), _native.ptr(offsets[b0:]),
                     _native.ptr(indices[b0:]), _native.ptr(ws), sz.value, stream)
        del cp, rows, vals
        if after_batch is not None:
            after_batch(b0 // tb)
    return matrices


def _finish_index(X, n_trees, depth, sparsity, seed, fixed_count, matrices, splits, offsets,
                  indices, checksum=None):
    Xd = X.device()
    sizes = offsets[:, 1:] - offsets[:, :-1]
    max_leaf = int(sizes.max().item())
    cp, rows, vals = _device.csc_device(matrices, pinned=True)
    dindex = _DeviceIndex(Xd, n_trees, depth, splits, offsets, indices, cp, rows, vals,
                          leaves_sorted=True, max_count=n_trees, max_leaf=max_leaf)
    # the streamed-vote layout is part of the index the queries use: built
    # here (billed to the build) wherever it applies
    dindex.vote_layout()
    return MRPTIndex(dataset=X, n_trees=n_trees, depth=depth, sparsity=float(sparsity), seed=seed,
                     fixed_count=fixed_count, matrices=matrices, splits=splits,
                     leaf_offsets=offsets, leaf_indices=indices,
                     dataset_checksum=checksum() if checksum else X.checksum,
                     _device_index=dindex)


def _alloc_index(n_trees, n, depth, dev):
    torch = _device.torch_mod()
    nleaf = 1 << depth
    return (torch.empty((n_trees, nleaf - 1), dtype=torch.float32, device=dev),
            torch.empty((n_trees, nleaf + 1), dtype=torch.int64, device=dev),
            torch.empty((n_trees, n), dtype=torch.int32, device=dev))


def grow_trees(X, n_trees, depth, sparsity=None, seed=0, fixed_count=False, threads=None,
               batch_trees=None):
    """Build ``n_trees`` trees of the given depth over ``X`` (trees.py:187-245).

    Same validation and errors as the reference.  ``threads`` (or
    MRPT_THREADS) is validated for compatibility; the work itself runs as
    batched GPU kernels.  ``batch_trees`` overrides the trees per launch.
    """
    X, sparsity, seed = _validate_grow(X, n_trees, depth, sparsity, seed, threads)
    checksum = X.checksum_async()  # K6 on a side stream, overlapping the build
    splits, offsets, indices = _alloc_index(n_trees, X.n, depth, X.device().device)
    matrices = _grow_block(X, 0, n_trees, depth, sparsity, seed, fixed_count, splits, offsets,
                           indices, batch_trees)
    return _finish_index(X, n_trees, depth, sparsity, seed, fixed_count, matrices, splits, offsets,
                         indices, checksum)
