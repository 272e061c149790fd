"""Query phase on the GPU (mirrors pkg/src/mrpt/search.py).

A query is projected onto every tree's matrix and descends to one leaf per
tree (K2, ``mrpt_query_route``); points sharing its leaf in at least
``votes`` trees are the candidates (K3, ``mrpt_vote``); the answer is the
exact float64 k-NN among them (K4, ``mrpt_scan_topk``).  The batched entry
point :func:`approximate_knn_batch` runs the three kernels over a whole
query matrix; the single-query functions keep the reference's signatures,
results and error order.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from . import _device, _native
from .core import _record_macs, as_dataset
from .exceptions import IntegrityError, ParameterError, ShapeError

__all__ = [
    "NeighborList",
    "VoteAccumulator",
    "approximate_knn",
    "approximate_knn_batch",
    "candidate_set",
    "exact_knn_in_set",
    "tree_query",
]


@dataclass(frozen=True)
class NeighborList:
    """Result of one query: ids by ascending distance, ties by ascending id
    (search.py:28-47)."""

    indices: np.ndarray  # int64
    distances: np.ndarray  # float64
    requested_k: int
    candidate_count: int

    def __len__(self):
        return int(self.indices.shape[0])

    @property
    def shortfall(self):
        return max(0, self.requested_k - len(self))


class VoteAccumulator:
    """Per-point vote counts of the last query (search.py:50-86), held on the GPU.

    ``accumulate`` counts every occurrence of every id in the given leaves
    (one per tree) and returns, ascending, the ids with at least ``votes``.
    Ascending is the order of the reference's numpy backend (``_py.vote``,
    _py.py:63-83); its compiled backend emits ids in threshold-crossing order
    (_cy.pyx:66-77), an order the reference's own tests do not rely on
    (test_kernels.py:59-78 compares the two backends as sets).  The set is
    identical; ``tests/test_gpu_reference_behaviour.py`` checks it against an
    unsorted list written by the compiled reference.
    """

    def __init__(self, n):
        self.n = n
        self._counts = None
        self._epoch = 0
        self._filled = -1  # epoch whose counts the device buffer holds

    def begin(self):
        self._epoch += 1
        return self._epoch

    def _buf(self):
        if self._counts is None:
            self._counts = _device.empty((self.n,), _device.torch_mod().int32)
        return self._counts

    def counts(self):
        """Dense n-vector of the current query's votes (int64 copy)."""
        # begin() starts a new epoch: like the reference's stamps (search.py:
        # 68-73), every count reads 0 until the next accumulate
        if self._counts is None or self._filled != self._epoch:
            return np.zeros(self.n, dtype=np.int64)
        return _device.d2h(self._counts).astype(np.int64)

    def count(self, i):
        if self._counts is None or self._filled != self._epoch:
            return 0
        return int(self._counts[int(i)].item())

    def accumulate(self, index, leaves, votes):
        torch = _device.torch_mod()
        self.begin()
        D = index.device_index()
        lv = leaves if _device.is_tensor(leaves) else _device.h2d(np.asarray(leaves, np.int32))
        lv = lv.to(torch.int32)
        counts = self._buf()
        stream = _native.stream_ptr()
        _native.call("mrpt_vote_counts", _native.ptr(D.indices), _native.ptr(D.offsets), D.n, D.T,
                     D.depth, _native.ptr(lv), _native.ptr(counts), stream)
        self._filled = self._epoch
        out = torch.empty(D.n, dtype=torch.int32, device=counts.device)
        nout = torch.zeros(1, dtype=torch.int64, device=counts.device)
        _native.call("mrpt_select_ge", _native.ptr(counts), D.n, int(votes), _native.ptr(out),
                     _native.ptr(nout), stream)
        return _device.d2h(out[:int(nout.item())]).astype(np.int64)


def _query_vector(q, d):
    arr = np.asarray(q)
    if arr.ndim != 1:
        raise ShapeError(f"query must be 1-D, got shape {arr.shape}")
    if arr.shape[0] != d:
        raise ShapeError(f"query has length {arr.shape[0]}, expected {d}")
    return np.ascontiguousarray(arr, dtype=np.float32)


def _route_device(Qd, D):
    """(nq, T) int32 leaves of a device query block (K2)."""
    torch = _device.torch_mod()
    nq = int(Qd.shape[0])
    leaves = torch.empty((nq, D.T), dtype=torch.int32, device=Qd.device)
    _native.call("mrpt_query_route", _native.ptr(Qd), nq, D.d, int(Qd.stride(0)),
                 _native.ptr(D.col_ptr), _native.ptr(D.rows), _native.ptr(D.vals),
                 _native.ptr(D.splits), D.T, D.depth, _native.ptr(leaves), _native.stream_ptr())
    return leaves


def _route_tree(q, tree):
    """Leaf id of ``q`` in one tree (search.py:100-102), on the device."""
    from .core import _project_device

    qd = _device.h2d(np.ascontiguousarray(q, dtype=np.float32).reshape(1, -1))
    _record_macs(tree.random_matrix.nnz)
    proj = _project_device(qd, tree.random_matrix)
    torch = _device.torch_mod()
    sp = _device.h2d(np.ascontiguousarray(tree.splits, dtype=np.float32).reshape(1, -1))
    out = torch.empty(1, dtype=torch.int64, device=qd.device)
    _native.call("mrpt_route", _native.ptr(proj), 1, tree.depth, _native.ptr(sp),
                 int(sp.shape[1]), _native.ptr(out), _native.stream_ptr())
    return int(out.item())


def tree_query(q, tree):
    """Point ids of the leaf ``q`` reaches in one tree (search.py:105-113)."""
    q = _query_vector(q, tree.random_matrix.d)
    return tree.leaf(_route_tree(q, tree))


def _accumulator(index):
    acc = getattr(index._local, "acc", None)
    if acc is None or acc.n != index.n:
        acc = index._local.acc = VoteAccumulator(index.n)
    return acc


def candidate_set(q, index, votes, accumulator=None):
    """Points sharing a leaf with ``q`` in at least ``votes`` trees, ascending,
    plus the accumulator holding all counts (search.py:130-143)."""
    if not 1 <= votes <= index.n_trees:
        raise ParameterError(f"vote threshold must lie in [1, {index.n_trees}], got {votes}")
    q = _query_vector(q, index.d)
    D = index.device_index()
    for R in index.matrices:
        _record_macs(R.nnz)
    leaves = _route_device(_device.h2d(q.reshape(1, -1)), D)[0]
    acc = accumulator if accumulator is not None else _accumulator(index)
    return acc.accumulate(index, leaves, votes), acc


def _topk_device(Xd, Qd, cand, cap, ncand, k):
    torch = _device.torch_mod()
    nq = int(Qd.shape[0])
    ids = torch.empty((nq, k), dtype=torch.int64, device=Qd.device)
    dists = torch.empty((nq, k), dtype=torch.float64, device=Qd.device)
    _native.call("mrpt_scan_topk", _native.ptr(Xd), int(Xd.shape[0]), int(Xd.shape[1]),
                 int(Xd.stride(0)), _native.ptr(Qd), nq, int(Qd.stride(0)), _native.ptr(cand),
                 int(cap), _native.ptr(ncand), int(k), _native.ptr(ids), _native.ptr(dists),
                 _native.stream_ptr())
    return ids, dists


def exact_knn_in_set(q, k, candidates, X):
    """Exact k-NN of ``q`` among ``candidates`` of ``X`` (search.py:146-172):
    duplicates collapsed, out-of-range ids rejected, float64 distances,
    (distance, id) order."""
    if k < 1:
        raise ParameterError(f"k must be >= 1, got {k}")
    X = as_dataset(X)
    q = _query_vector(q, X.d)
    torch = _device.torch_mod()
    c = np.asarray(candidates, dtype=np.int64).ravel()
    if c.shape[0] == 0:
        return NeighborList(indices=np.empty(0, np.int64), distances=np.empty(0, np.float64),
                            requested_k=k, candidate_count=0)
    Xd = X.device()
    cd = _device.h2d(c)
    bitmap = torch.empty((X.n + 31) // 32, dtype=torch.int32, device=Xd.device)
    uniq = torch.empty(min(X.n, c.shape[0]) + 1, dtype=torch.int32, device=Xd.device)
    nout = torch.zeros(1, dtype=torch.int64, device=Xd.device)
    bad = torch.zeros(1, dtype=torch.int32, device=Xd.device)
    stream = _native.stream_ptr()
    _native.call("mrpt_unique_ids", _native.ptr(cd), c.shape[0], X.n, _native.ptr(bitmap),
                 _native.ptr(uniq), _native.ptr(nout), _native.ptr(bad), stream)
    if int(bad.item()):
        raise IntegrityError(f"candidate indices must lie in [0, {X.n}), got range "
                             f"[{int(c.min())}, {int(c.max())}]")
    ncand = nout.to(torch.int32)
    m = int(nout.item())
    ids, dists = _topk_device(Xd, _device.h2d(q.reshape(1, -1)), uniq, uniq.shape[0], ncand, k)
    kept = min(k, m)
    return NeighborList(indices=_device.d2h(ids[0, :kept]), distances=_device.d2h(dists[0, :kept]),
                        requested_k=k, candidate_count=m)


def _check_batch_args(k, index, votes):
    if k < 1:
        raise ParameterError(f"k must be >= 1, got {k}")
    if not 1 <= votes <= index.n_trees:
        raise ParameterError(f"vote threshold must lie in [1, {index.n_trees}], got {votes}")


def _chunk_bytes():
    """Scratch (leaves + candidate lists) of one query chunk of a batch."""
    return int(os.environ.get("MRPT_CHUNK_BYTES", 1 << 30))


def query_device(D, Qd, k, votes, chunk=None, out=None, timer=None, size_class=None):
    """K2 -> K3 -> K4 over a device query block; returns device tensors
    (ids (nq,k) int64, dists (nq,k) float64, candidate_count (nq,) int32).
    ``timer``: optional list receiving (stage, start_event, end_event) per launch.
    The candidate hand-over is a list per query, or a bitmap per query for
    the GEMM filter when the autotune found that faster (both exact)."""
    torch = _device.torch_mod()

    def stage(name, fn, *a):
        if timer is None:
            return fn(*a)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(*a)
        e1.record()
        timer.append((name, e0, e1))

    nq = int(Qd.shape[0])
    dev = Qd.device
    cap = D.cap(votes)
    if out is None:
        ids = torch.empty((nq, k), dtype=torch.int64, device=dev)
        dists = torch.empty((nq, k), dtype=torch.float64, device=dev)
        counts = torch.empty(nq, dtype=torch.int32, device=dev)
    else:
        ids, dists, counts = out
    bstride = _bstride(D)
    # the route is chosen per batch-size class of this call (the caller's
    # class when this is the rest of an autotuned batch)
    sc = _size_class(int(Qd.shape[0])) if size_class is None else size_class
    choice = D.scan_pin.get((k, votes)) or D.scan_choice_by_size.get((k, votes, sc))
    bits_mode = choice in _BITS_ROUTES
    if chunk is None:
        per_q = 4 * (D.T + (bstride if bits_mode else cap))
        chunk = max(1, min(nq, _chunk_bytes() // per_q))
        # whole waves: the vote runs one CTA per SM and the filters up to four,
        # each CTA striding over the chunk's queries
        wave = 4 * _device.sm_count()
        if wave < chunk < nq and os.environ.get("MRPT_CHUNK_WAVES", "1") != "0":
            chunk -= chunk % wave  # (a batch that fits one chunk stays one chunk)
    if (not bits_mode and choice is not None and nq >= 2 * _ORDER_MIN
            and os.environ.get("MRPT_QUERY_ORDER", "1") != "0" and D.vote_layout() is not None
            and nq * D.T * 4 <= (2 << 30)):
        return _query_device_ordered(D, Qd, k, votes, choice, cap, chunk, stage, (ids, dists, counts))
    m0 = min(chunk, nq)
    leaves = torch.empty((m0, D.T), dtype=torch.int32, device=dev)
    cand = None
    bits = torch.empty((m0, bstride), dtype=torch.int32, device=dev) if bits_mode else None
    for s in range(0, nq, chunk):
        e = min(nq, s + chunk)
        qb = Qd[s:e]
        if bits_mode:
            _run_bits(D, qb, e - s, int(Qd.stride(0)), leaves, votes, bits, bstride,
                      counts[s:e], k, ids[s:e], dists[s:e], stage, route=choice)
            continue
        stage("route", _route_launch, D, qb, e - s, int(Qd.stride(0)), leaves)
        if choice is None and e - s >= 256:
            # the autotune's last run leaves this chunk's outputs; the rest of
            # the batch runs the chosen route (its own chunking)
            _autotune(D, qb, e - s, int(Qd.stride(0)), leaves, votes, cap, counts[s:e], k, sc,
                      ids[s:e], dists[s:e])
            if e < nq:
                query_device(D, Qd[e:], k, votes, out=(ids[e:], dists[e:], counts[e:]), timer=timer,
                             size_class=sc)
            return ids, dists, counts
        if cand is None:
            cand = torch.empty((m0, cap), dtype=torch.int32, device=dev)
        stage("vote", _vote_list, D, leaves, e - s, votes, cand, cap, counts[s:e])
        args = (qb, e - s, int(Qd.stride(0)), cand, cap, counts[s:e], k, ids[s:e], dists[s:e])
        variant = choice if choice is not None and choice not in _BITS_ROUTES else "fp32"
        if choice is None:  # small batch, no autotune: a forced list route still applies
            env = os.environ.get("MRPT_SCAN_ROWS")
            if env and env not in _BITS_ROUTES and env in _scan_variants(D, k):
                variant = env
        stage("scan_topk", _scan_launch, D, variant, args)
    return ids, dists, counts


_BITS_ROUTES = ("u8tc_bits",)
_ORDER_MIN = 4096  # queries: below this a batch is processed in its own order
_order_hook = None  # experiments (tools/order_ab.py): callable(leaves, Qd) -> int32 query order


def _permute(src, idx, dst, scatter):
    """dst[i] = src[idx[i]] (gather) or dst[idx[i]] = src[i] (scatter), rows of
    4-byte words (mrpt_permute_rows)."""
    words = src[0].numel() * src.element_size() // 4
    _native.call("mrpt_permute_rows", _native.ptr(src), int(src.stride(0)) * src.element_size() // 4,
                 _native.ptr(idx), int(idx.shape[0]), words, _native.ptr(dst),
                 int(dst.stride(0)) * dst.element_size() // 4, 1 if scatter else 0,
                 _native.stream_ptr())


def _query_device_ordered(D, Qd, k, votes, variant, cap, chunk, stage, out):
    """query_device for a large batch over a multi-tile index: route the whole
    batch (K2), order the queries by their leaf in tree 0
    (mrpt_query_order), gather the query rows and leaves into that order, run
    K3 + K4 chunk by chunk on the ordered batch -- concurrent CTAs then share
    leaf slices and candidate rows in L2 -- and scatter the answers back.
    Identical results (queries are independent)."""
    torch = _device.torch_mod()
    nq = int(Qd.shape[0])
    dev = Qd.device
    leaves = torch.empty((nq, D.T), dtype=torch.int32, device=dev)
    stage("route", _route_launch, D, Qd, nq, int(Qd.stride(0)), leaves)
    order = torch.empty(nq, dtype=torch.int32, device=dev)
    ws = D.workspace("qorder", 4 << D.depth)
    Qp = torch.empty((nq, D.d), dtype=torch.float32, device=dev)
    lp = torch.empty_like(leaves)

    def reorder():
        if _order_hook is not None:
            order.copy_(_order_hook(leaves, Qd))
        else:
            _native.call("mrpt_query_order", _native.ptr(leaves), nq, D.T, D.depth, _native.ptr(order),
                         _native.ptr(ws), _native.stream_ptr())
        _permute(Qd, order, Qp, False)
        _permute(leaves, order, lp, False)

    stage("reorder", reorder)
    ids = torch.empty((nq, k), dtype=torch.int64, device=dev)
    dists = torch.empty((nq, k), dtype=torch.float64, device=dev)
    counts = torch.empty(nq, dtype=torch.int32, device=dev)
    m0 = min(chunk, nq)
    cand = torch.empty((m0, cap), dtype=torch.int32, device=dev)
    for s in range(0, nq, chunk):
        e = min(nq, s + chunk)
        stage("vote", _vote_list, D, lp[s:e], e - s, votes, cand, cap, counts[s:e])
        args = (Qp[s:e], e - s, int(Qp.stride(0)), cand, cap, counts[s:e], k, ids[s:e], dists[s:e])
        stage("scan_topk", _scan_launch, D, variant, args)
    oids, odists, ocounts = out

    def restore():
        _permute(ids, order, oids, True)
        _permute(dists, order, odists, True)
        _permute(counts.view(nq, 1), order, ocounts.view(nq, 1), True)

    stage("reorder", restore)
    return oids, odists, ocounts


def _run_bits(D, qb, m, ldq, leaves, votes, bits, bstride, counts, k, ids, dists, stage=None,
              route="u8tc_bits"):
    """The bitmap route: K2 + K3 on their own stream beside K4's query
    quantisation, which needs only the queries; the fused tcgen05 filter
    waits for the candidate bitmaps."""
    torch = _device.torch_mod()
    if stage is None:
        def stage(name, fn, *a):
            fn(*a)
    vs = _device.vote_stream()
    ev_start = torch.cuda.Event()
    ev_start.record()
    with torch.cuda.stream(vs):
        vs.wait_event(ev_start)
        stage("route", _route_launch, D, qb, m, ldq, leaves)
        stage("vote", _vote_bitmap, D, leaves, m, votes, bits, bstride, counts)
        ev_vote = torch.cuda.Event()
        ev_vote.record(vs)
    stage("scan_topk", _scan_tc, D, qb, m, ldq, bits, bstride, k, ids, dists, ev_vote)
    torch.cuda.current_stream().wait_event(ev_vote)  # leaves/bits are reused


def _bstride(D):
    """Words per query of a candidate bitmap (16-byte rows)."""
    return (D.n + 127) // 128 * 4


def _route_launch(D, qb, m, ldq, leaves):
    _native.call("mrpt_query_route", _native.ptr(qb), m, D.d, int(ldq), _native.ptr(D.col_ptr),
                 _native.ptr(D.rows), _native.ptr(D.vals), _native.ptr(D.splits), D.T, D.depth,
                 _native.ptr(leaves), _native.stream_ptr())


def _vote_list(D, leaves, m, votes, cand, cap, counts):
    lay = D.vote_layout()
    if lay == "pair" and votes <= D.pair_max_votes():
        # the paired streamed vote (two id tiles per load, second parked in TMEM;
        # saturating 8-bit counters when T > 255, which bound the threshold --
        # larger thresholds take mrpt_vote below)
        ps, pstride, pdir, pbase = D.vote_pair()
        _native.call("mrpt_vote_pair", _native.ptr(ps), int(pstride), _native.ptr(pdir),
                     _native.ptr(pbase), D.n, D.T, D.depth, int(D.max_count), _native.ptr(leaves), m,
                     int(votes), _native.ptr(cand), int(cap), _native.ptr(counts),
                     _native.stream_ptr())
        return
    vs = D.vote_stream() if lay == "stream" else None
    if vs is not None:
        # the streamed tiled vote (padded, pre-decoded leaf slices)
        qs, tstride, qdir, qbase = vs
        _native.call("mrpt_vote_stream", _native.ptr(qs), int(tstride), _native.ptr(qdir),
                     _native.ptr(qbase), D.n, D.T, D.depth, int(D.max_count), _native.ptr(leaves), m,
                     int(votes), _native.ptr(cand), int(cap), _native.ptr(counts),
                     _native.stream_ptr())
        return
    _native.call("mrpt_vote", _native.ptr(D.indices), _native.ptr(D.offsets), D.n, D.T, D.depth,
                 _native.ptr(leaves), m, int(votes), int(D.leaves_sorted), int(D.max_count),
                 _native.ptr(D.vote_dir()), _native.ptr(cand), int(cap), _native.ptr(counts),
                 _native.stream_ptr())


def _vote_bitmap(D, leaves, m, votes, bits, bstride, counts):
    _native.call("mrpt_vote_bitmap", _native.ptr(D.indices), _native.ptr(D.offsets), D.n, D.T,
                 D.depth, _native.ptr(leaves), m, int(votes), int(D.leaves_sorted),
                 int(D.max_count), _native.ptr(D.vote_dir()), _native.ptr(bits), int(bstride),
                 _native.ptr(counts), _native.stream_ptr())


def _scan_tc(D, qb, m, ldq, bits, bstride, k, ids, dists, wait=None):
    ldr = D.u8_rows()[1]
    Xs, info, ws = D.u8_tc(m)
    _native.call("mrpt_scan_topk_u8tc_bits", _native.ptr(D.X), D.n, D.d, int(D.X.stride(0)),
                 _native.ptr(Xs), ldr, _native.ptr(info), _native.ptr(qb), m, ldq,
                 _native.ptr(bits), int(bstride), int(k), _native.ptr(ids), _native.ptr(dists),
                 _native.ptr(ws), int(ws.numel()), None if wait is None else wait.cuda_event,
                 _native.stream_ptr())


def _scan_variants(D, k):
    """Exact filter variants available for this index (all give identical results)."""
    out = []
    if k <= 120 and D.u8_rows() is not None:
        out.append("u8")
        # the fused tcgen05 filter over K3's bitmaps: one 128-B K block at
        # least, the queries' k smallest bounds in shared memory (k <= 16),
        # 16-byte rows for its exact fallback, bitmaps of at most 4M ids
        aligned = D.d % 4 == 0 and int(D.X.stride(0)) % 4 == 0 and D.X.data_ptr() % 16 == 0
        if k <= 16 and aligned and 128 <= D.u8_rows()[1] <= 1024 and D.n <= (4 << 20):
            out.append("u8tc_bits")
    if k <= 120 and D.shadow() is not None:
        out.append("fp16")
    out.append("fp32")
    return out


def _scan_launch(D, variant, args):
    """K4 over one query chunk with the chosen filter rows."""
    qb, m, ldq, cand, cap, counts, k, ids, dists = args
    stream = _native.stream_ptr()
    common_tail = (_native.ptr(qb), m, ldq, _native.ptr(cand), int(cap), _native.ptr(counts),
                   int(k), _native.ptr(ids), _native.ptr(dists), stream)
    if variant == "u8":
        Xq, ldr, sc, nm, rad = D.u8_rows()
        _native.call("mrpt_scan_topk_u8", _native.ptr(D.X), D.n, D.d, int(D.X.stride(0)),
                     _native.ptr(Xq), ldr, _native.ptr(sc), _native.ptr(nm), _native.ptr(rad),
                     *common_tail)
    elif variant == "fp16":
        Xh, ldh, rad = D.shadow()
        _native.call("mrpt_scan_topk_fp16", _native.ptr(D.X), D.n, D.d, int(D.X.stride(0)),
                     _native.ptr(Xh), ldh, _native.ptr(rad), *common_tail)
    else:
        _native.call("mrpt_scan_topk", _native.ptr(D.X), D.n, D.d, int(D.X.stride(0)),
                     *common_tail)


def _autotune(D, qb, m, ldq, leaves, votes, cap, counts, k, sc, ids, dists):
    """Time every exact route for this chunk -- list vote + each list filter,
    bitmap vote + the fused tcgen05 filter -- and keep the fastest for the index
    (per k and vote threshold); the last run leaves valid outputs (all routes
    give identical results).  MRPT_SCAN_ROWS forces a variant."""
    torch = _device.torch_mod()
    variants = _scan_variants(D, k)
    env = os.environ.get("MRPT_SCAN_ROWS")
    if env in variants:
        variants = [env]
    dev = qb.device
    list_vars = [v for v in variants if v not in _BITS_ROUTES]
    times = {}

    def timed(fn, *a):
        fn(*a)  # warm (first use builds the filter rows)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(*a)
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1)

    tr = timed(_route_launch, D, qb, m, ldq, leaves)
    for route in _BITS_ROUTES:
        if route not in variants:
            continue
        # timed as it runs: route + vote beside the quantisation (and GEMM),
        # then the filter
        bstride = _bstride(D)
        bits = torch.empty((m, bstride), dtype=torch.int32, device=dev)
        times[route] = timed(_run_bits, D, qb, m, ldq, leaves, votes, bits, bstride,
                             counts, k, ids, dists, None, route)
    if list_vars:
        cand = torch.empty((m, cap), dtype=torch.int32, device=dev)
        tv = tr + timed(_vote_list, D, leaves, m, votes, cand, cap, counts)
        args = (qb, m, ldq, cand, cap, counts, k, ids, dists)
        for v in list_vars:
            times[v] = tv + timed(_scan_launch, D, v, args)
    best = min(times, key=times.get)
    D.scan_choice[(k, votes)] = best
    D.scan_choice_by_size[(k, votes, sc)] = best
    return best


def _size_class(m):
    """Batch-size class of the per-index route autotune: the routes' relative
    speed depends on how many queries share one launch (the fused tcgen05
    filter needs many query blocks per CTA)."""
    c = 0
    while c < 3 and m >= (2048 << c):
        c += 1
    return c


def approximate_knn_batch(Q, k, index, votes, chunk=None):
    """Approximate k-NN for every row of ``Q`` in one batched GPU pass.

    Returns (ids int64 (nq, k) padded with -1, dists float64 (nq, k) padded
    with +inf, candidate_count int32 (nq,)).  Host input gives host arrays;
    a CUDA tensor gives CUDA tensors and nothing is synchronised.
    Row i equals ``approximate_knn(Q[i], k, index, votes)`` exactly.
    """
    _check_batch_args(k, index, votes)
    on_device = _device.is_tensor(Q) and Q.is_cuda
    torch = _device.torch_mod()
    if not on_device and chunk is None:
        Qc = Q if _device.is_tensor(Q) else None
        if Qc is None:
            Qh = np.asarray(Q)
            if Qh.ndim == 2 and Qh.shape[1] == index.d and Qh.shape[0] >= 2 * _PIPE_MIN:
                Qc = torch.from_numpy(np.ascontiguousarray(Qh, dtype=np.float32))
        if Qc is not None and Qc.dim() == 2 and Qc.shape[1] == index.d and Qc.shape[0] >= 2 * _PIPE_MIN:
            return _knn_batch_pipelined(Qc, k, index, votes)
    if _device.is_tensor(Q):
        if Q.dim() != 2 or Q.shape[1] != index.d:
            raise ShapeError(f"queries must be (nq, {index.d}), got {tuple(Q.shape)}")
        # a pinned host tensor is copied asynchronously on the current stream
        Qd = Q.to(device=_device.device(), dtype=torch.float32,
                  non_blocking=True).contiguous()
    else:
        Qh = np.asarray(Q)
        if Qh.ndim != 2 or Qh.shape[1] != index.d:
            raise ShapeError(f"queries must be (nq, {index.d}), got {Qh.shape}")
        Qd = _device.h2d(np.ascontiguousarray(Qh, dtype=np.float32))
    D = index.device_index()
    nq = int(Qd.shape[0])
    nnz = sum(R.nnz for R in index.matrices)
    _record_macs(nq * nnz)
    if nq == 0:
        z = (np.empty((0, k), np.int64), np.empty((0, k), np.float64), np.empty(0, np.int32))
        return z
    ids, dists, counts = query_device(D, Qd, k, votes, chunk=chunk)
    if on_device:
        return ids, dists, counts
    return _device.d2h(ids), _device.d2h(dists), _device.d2h(counts)


_PIPE_MIN = 2048  # queries per pipelined piece (at least)


def _pipe_bounds(nq, mode=""):
    """Piece boundaries of a pipelined host batch: a small first piece (its
    upload is the only one not hidden under compute), then a larger
    one (MRPT_PIPE_REST pieces, default 1: the fused filter wants full
    launches).  mode "equal": up to 4 equal pieces."""
    if mode == "equal":
        pieces = max(1, min(4, nq // _PIPE_MIN))
        return [nq * i // pieces for i in range(pieces + 1)]
    if mode == "one":
        return [0, nq]
    if mode.startswith("first"):  # "firstN": a first piece of N queries, then the rest
        first = min(nq, max(1, int(mode[5:])))
        return [0, first, nq] if first < nq else [0, nq]
    first = min(nq, max(256, nq // 8))
    rest = nq - first
    pieces = max(1, min(int(os.environ.get("MRPT_PIPE_REST", "1")), rest // _PIPE_MIN))
    return [0] + [first + rest * i // pieces for i in range(pieces + 1)]


def _knn_batch_pipelined(Qc, k, index, votes):
    """Host queries in, host results out, with the transfers overlapped: the
    batch is cut into up to 4 pieces; piece i's upload (copy stream), its
    route/vote/scan (compute stream, after the upload's event) and its
    results' download into pinned host memory (a third stream, after the
    compute event) are enqueued in that order, so uploads of later pieces and
    downloads of earlier ones run under the compute of the others.  Results
    are identical to the unpipelined path."""
    torch = _device.torch_mod()
    D = index.device_index()
    nq = int(Qc.shape[0])
    Qc = Qc.to(dtype=torch.float32).contiguous()
    _record_macs(nq * sum(R.nnz for R in index.matrices))
    route = D.scan_pin.get((k, votes)) or D.scan_choice_by_size.get((k, votes, _size_class(nq)))
    if route in _BITS_ROUTES and not os.environ.get("MRPT_PIPE") and \
            4 * nq * (D.T + _bstride(D)) <= (1 << 30):
        return _knn_batch_pipelined_bits(Qc, k, index, votes, route)
    bounds = _pipe_bounds(nq, os.environ.get("MRPT_PIPE", ""))
    pieces = len(bounds) - 1
    dev = _device.device()
    Qd = torch.empty((nq, index.d), dtype=torch.float32, device=dev)
    ids = torch.empty((nq, k), dtype=torch.int64, device=dev)
    dists = torch.empty((nq, k), dtype=torch.float64, device=dev)
    counts = torch.empty(nq, dtype=torch.int32, device=dev)
    hid = torch.empty((nq, k), dtype=torch.int64, pin_memory=True)
    hdist = torch.empty((nq, k), dtype=torch.float64, pin_memory=True)
    hcnt = torch.empty(nq, dtype=torch.int32, pin_memory=True)
    compute = torch.cuda.current_stream()
    up, down = _device.side_streams()
    # Qd came from the caching allocator on the compute stream: work still
    # queued there may own that block, so the uploads wait for it first
    up.wait_stream(compute)
    for i in range(pieces):
        s, e = bounds[i], bounds[i + 1]
        with torch.cuda.stream(up):
            Qd[s:e].copy_(Qc[s:e], non_blocking=True)
            ev_up = torch.cuda.Event()
            ev_up.record(up)
        compute.wait_event(ev_up)
        query_device(D, Qd[s:e], k, votes, out=(ids[s:e], dists[s:e], counts[s:e]))
        ev_done = torch.cuda.Event()
        ev_done.record(compute)
        with torch.cuda.stream(down):
            down.wait_event(ev_done)
            hid[s:e].copy_(ids[s:e], non_blocking=True)
            hdist[s:e].copy_(dists[s:e], non_blocking=True)
            hcnt[s:e].copy_(counts[s:e], non_blocking=True)
    down.synchronize()  # after every piece's compute and upload, too
    return hid.numpy(), hdist.numpy(), hcnt.numpy()


def _knn_batch_pipelined_bits(Qc, k, index, votes, route):
    """Host batch over a bitmap route: the upload is cut into pieces and each
    piece's route + vote (K2 + K3, bitmaps into one batch-wide buffer) runs
    as soon as it lands, under the next piece's upload; then ONE filter
    launch covers the whole batch (the fused filter wants full launches), and
    the results come back in one download.  Results are identical."""
    torch = _device.torch_mod()
    D = index.device_index()
    nq = int(Qc.shape[0])
    dev = _device.device()
    bstride = _bstride(D)
    Qd = torch.empty((nq, index.d), dtype=torch.float32, device=dev)
    leaves = torch.empty((nq, D.T), dtype=torch.int32, device=dev)
    bits = torch.empty((nq, bstride), dtype=torch.int32, device=dev)
    ids = torch.empty((nq, k), dtype=torch.int64, device=dev)
    dists = torch.empty((nq, k), dtype=torch.float64, device=dev)
    counts = torch.empty(nq, dtype=torch.int32, device=dev)
    hid = torch.empty((nq, k), dtype=torch.int64, pin_memory=True)
    hdist = torch.empty((nq, k), dtype=torch.float64, pin_memory=True)
    hcnt = torch.empty(nq, dtype=torch.int32, pin_memory=True)
    compute = torch.cuda.current_stream()
    up, _ = _device.side_streams()
    up.wait_stream(compute)  # Qd's block may still be in use by queued compute work
    pieces = max(1, min(int(os.environ.get("MRPT_PIPE_PIECES", "4")), nq // 1024))
    bounds = [nq * i // pieces for i in range(pieces + 1)]
    for i in range(pieces):
        s, e = bounds[i], bounds[i + 1]
        with torch.cuda.stream(up):
            Qd[s:e].copy_(Qc[s:e], non_blocking=True)
            ev_up = torch.cuda.Event()
            ev_up.record(up)
        compute.wait_event(ev_up)
        _route_launch(D, Qd[s:e], e - s, int(Qd.stride(0)), leaves[s:e])
        _vote_bitmap(D, leaves[s:e], e - s, votes, bits[s:e], bstride, counts[s:e])
    _scan_tc(D, Qd, nq, int(Qd.stride(0)), bits, bstride, k, ids, dists)
    hid.copy_(ids, non_blocking=True)
    hdist.copy_(dists, non_blocking=True)
    hcnt.copy_(counts, non_blocking=True)
    compute.synchronize()
    return hid.numpy(), hdist.numpy(), hcnt.numpy()


_SWEEP_SCRATCH_BYTES = 1 << 30  # leaves + candidates + counts of one sweep chunk


def approximate_knn_sweep(Q, k, index, votes):
    """approximate_knn_batch for several vote thresholds from ONE route and
    ONE vote pass (the reference's sweeps loop queries and
    thresholds one at a time, evaluation.py:163-215): the vote at the smallest
    threshold also records each candidate's count, every larger threshold
    filters that list (counts do not depend on v), and each threshold's
    candidates go through the exact scan.  Returns {v: (ids, dists, counts)}
    with host arrays for host input, CUDA tensors for a CUDA tensor; each
    entry equals approximate_knn_batch(Q, k, index, v)."""
    vs = sorted({int(v) for v in votes})
    if not vs:
        return {}
    for v in vs:
        _check_batch_args(k, index, v)
    torch = _device.torch_mod()
    on_device = _device.is_tensor(Q) and Q.is_cuda
    if _device.is_tensor(Q):
        Qd = Q.to(device=_device.device(), dtype=torch.float32).contiguous()
    else:
        Qd = _device.h2d(np.ascontiguousarray(np.asarray(Q), dtype=np.float32))
    if Qd.dim() != 2 or Qd.shape[1] != index.d:
        raise ShapeError(f"queries must be (nq, {index.d}), got {tuple(Qd.shape)}")
    D = index.device_index()
    nq = int(Qd.shape[0])
    dev = Qd.device
    _record_macs(nq * sum(R.nnz for R in index.matrices) * len(vs))
    cap0 = D.cap(vs[0])
    # query rows go through in chunks sized like query_device's (1 GiB of
    # leaves + candidate + count scratch), so a batch that approximate_knn_batch
    # answers never runs out of memory here
    rows = max(1, min(max(1, nq), _SWEEP_SCRATCH_BYTES // (4 * D.T + 6 * cap0)))
    leaves = torch.empty((rows, D.T), dtype=torch.int32, device=dev)
    cand0 = torch.empty((rows, cap0), dtype=torch.int32, device=dev)
    cnt0 = torch.empty((rows, cap0), dtype=torch.int16, device=dev)
    n0 = torch.empty(rows, dtype=torch.int32, device=dev)
    res = {v: (torch.empty((nq, k), dtype=torch.int64, device=dev),
               torch.empty((nq, k), dtype=torch.float64, device=dev),
               torch.empty(nq, dtype=torch.int32, device=dev)) for v in vs}
    caps = {v: D.cap(v) for v in vs}
    cands = {v: torch.empty((rows, caps[v]), dtype=torch.int32, device=dev) for v in vs[1:]}
    for lo in range(0, nq, rows):
        m = min(rows, nq - lo)
        Qc = Qd[lo:lo + m]
        _route_launch(D, Qc, m, int(Qd.stride(0)), leaves)
        _native.call("mrpt_vote_counted", _native.ptr(D.indices), _native.ptr(D.offsets), D.n, D.T,
                     D.depth, _native.ptr(leaves), m, vs[0], int(D.leaves_sorted),
                     int(D.max_count), _native.ptr(D.vote_dir()), _native.ptr(cand0),
                     _native.ptr(cnt0), int(cap0), _native.ptr(n0), _native.stream_ptr())
        for v in vs:
            ids, dists, counts_all = res[v]
            counts = counts_all[lo:lo + m]
            if v == vs[0]:
                cand, cap = cand0, cap0
                counts.copy_(n0[:m])
            else:
                cand, cap = cands[v], caps[v]
                _native.call("mrpt_filter_counts", _native.ptr(cand0), _native.ptr(cnt0), int(cap0),
                             _native.ptr(n0), m, v, _native.ptr(cand), int(cap),
                             _native.ptr(counts), _native.stream_ptr())
            variant = D.scan_choice.get((k, v))
            if variant is None or variant in _BITS_ROUTES:
                variant = [x for x in _scan_variants(D, k) if x not in _BITS_ROUTES][0]
            args = (Qc, m, int(Qd.stride(0)), cand, cap, counts, k, ids[lo:lo + m], dists[lo:lo + m])
            _scan_launch(D, variant, args)
    out = {v: (r if on_device else tuple(_device.d2h(t) for t in r)) for v, r in res.items()}
    return out


def approximate_knn(q, k, index, votes):
    """Approximate k-NN of one query (search.py:175-184): vote-filtered
    candidates, then the exact scan; ``shortfall`` reports a deficit."""
    if k < 1:
        raise ParameterError(f"k must be >= 1, got {k}")
    if not 1 <= votes <= index.n_trees:
        raise ParameterError(f"vote threshold must lie in [1, {index.n_trees}], got {votes}")
    q = _query_vector(q, index.d)
    ids, dists, counts = approximate_knn_batch(q.reshape(1, -1), k, index, votes)
    m = int(counts[0])
    kept = min(k, m)
    return NeighborList(indices=ids[0, :kept].copy(), distances=dists[0, :kept].copy(),
                        requested_k=k, candidate_count=m)


def vote_stats(reset=False):
    """Saturating paired vote (8-bit counters with T > 255): queries voted
    and queries redone exactly after a counter wrapped, since the last reset
    (measurement; synchronises the device)."""
    import ctypes

    out = (ctypes.c_int64 * 2)()
    _native.call("mrpt_vote_stats", out, 1 if reset else 0)
    return {"queries": int(out[0]), "redone": int(out[1])}


def fallback_stats(reset=False):
    """How often each exact filter route handed queries to its exact tiled
    fallback since the last reset (measurement; synchronises the device):
    {route: {"queries": q, "fallbacks": f}} for fp32, fp16, u8, u8tc_bits."""
    import ctypes

    out = (ctypes.c_int64 * 8)()
    _native.call("mrpt_fallback_stats", out, 1 if reset else 0)
    names = ("fp32", "fp16", "u8", "u8tc_bits")
    return {nm: {"queries": int(out[2 * i]), "fallbacks": int(out[2 * i + 1])}
            for i, nm in enumerate(names)}
