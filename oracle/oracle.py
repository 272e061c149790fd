"""CPU oracle for the MRPT hot path -- TEST INFRASTRUCTURE ONLY.

A restatement of the reference algorithm (arXiv 1509.06957, /root/reference/pkg)
in numpy + the plain C kernels of ``mrpt_oracle.c``.  It is the parity checker
for the CUDA implementation: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / reference legs may import it, never the product.

Pinned against the reference itself: ``tests/golden/*.npz`` were produced by
the unmodified reference package (``tests/golden/make_golden.py``) and
``tests/test_oracle_golden.py`` checks this module against them bit for bit.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


def build():
    """Compile liboracle.so (gcc) if it is missing or stale."""
    so = os.path.join(HERE, "liboracle.so")
    src = os.path.join(HERE, "mrpt_oracle.c")
    if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", HERE, "liboracle.so"])
    return so


def lib():
    global _LIB
    if _LIB is None:
        L = ctypes.CDLL(build())
        c_i64, c_i32 = ctypes.c_int64, ctypes.c_int32
        L.oracle_project.argtypes = [_f32p, c_i64, c_i32, _i64p, _i32p, _f32p, c_i32, _f32p]
        L.oracle_route.argtypes = [_f32p, c_i64, c_i32, _f32p, c_i64, _i64p]
        L.oracle_build_tree.argtypes = [_f32p, c_i64, c_i32, c_i32, _f32p, _i64p, _i32p]
        L.oracle_vote_counts.argtypes = [_i32p, _i64p, c_i64, c_i32, c_i64, _i64p, _i32p]
        L.oracle_scan.argtypes = [_f32p, c_i32, _i64p, c_i64, _f32p, _f64p]
        L.oracle_fnv1a64.argtypes = [_u8p, c_i64]
        L.oracle_fnv1a64.restype = ctypes.c_uint64
        for f in ("oracle_project", "oracle_route", "oracle_build_tree", "oracle_vote_counts",
                  "oracle_scan"):
            getattr(L, f).restype = None
        _LIB = L
    return _LIB


# --- sampling: core.sample_sparse_matrix (pkg/src/mrpt/core.py:145-185) ------
def sample_sparse_matrix(d, depth, a, seed, fixed_count=False):
    """(col_ptr i64, row_idx i32, values f32) of the reference's matrix.

    Same Philox(SeedSequence(entropy)) stream, consumed in the same order:
    all Bernoulli gates (C order of a d x depth array) or, with fixed_count,
    one sorted choice per column; then the normals column by column, drawn in
    float64 and cast to float32 (core.py:159-179).
    """
    entropy = tuple(int(s) for s in seed) if isinstance(seed, (tuple, list)) else (int(seed),)
    gen = np.random.Generator(np.random.Philox(np.random.SeedSequence(entropy)))
    if fixed_count:
        per_col = math.ceil(a * d)
        cols = [np.sort(gen.choice(d, size=per_col, replace=False)) for _ in range(depth)]
    else:
        gate = gen.random((d, depth)) < a
        cols = [np.nonzero(gate[:, j])[0] for j in range(depth)]
    sizes = np.array([c.size for c in cols], dtype=np.int64)
    col_ptr = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    nnz = int(col_ptr[-1])
    row_idx = np.concatenate(cols).astype(np.int32) if nnz else np.zeros(0, np.int32)
    values = np.zeros(nnz, dtype=np.float32)
    for j in range(depth):
        values[col_ptr[j]:col_ptr[j + 1]] = gen.standard_normal(int(sizes[j]))
    return col_ptr, row_idx, values


# --- kernels -------------------------------------------------------------------
def project(X, col_ptr, row_idx, values):
    X = np.ascontiguousarray(X, dtype=np.float32)
    m, d = X.shape
    ncols = len(col_ptr) - 1
    out = np.empty((m, ncols), dtype=np.float32)
    lib().oracle_project(X, m, d, np.ascontiguousarray(col_ptr, np.int64),
                         np.ascontiguousarray(row_idx, np.int32),
                         np.ascontiguousarray(values, np.float32), ncols, out)
    return out


def route(proj, splits):
    proj = np.ascontiguousarray(proj, np.float32)
    splits = np.ascontiguousarray(splits, np.float32)
    out = np.empty(proj.shape[0], dtype=np.int64)
    lib().oracle_route(proj, proj.shape[0], proj.shape[1], splits, splits.shape[1], out)
    return out


def build_tree(P, depth):
    """(splits f32[2^depth-1], offsets i64[2^depth+1], order i32[n]) of trees.py:54-98."""
    P = np.ascontiguousarray(P, np.float32)
    n = P.shape[0]
    splits = np.zeros((1 << depth) - 1, dtype=np.float32)
    offsets = np.zeros((1 << depth) + 1, dtype=np.int64)
    order = np.zeros(n, dtype=np.int32)
    lib().oracle_build_tree(P, n, P.shape[1], depth, splits, offsets, order)
    return splits, offsets, order


def build_one_tree(X, depth, a, seed, t, fixed_count=False):
    """Tree t of grow_trees (trees.py:217-224): R from (seed, t), P = X R, build."""
    R = sample_sparse_matrix(X.shape[1], depth, a, (seed, t), fixed_count)
    P = project(X, *R)
    return R, build_tree(P, depth)


def grow_trees(X, n_trees, depth, a=None, seed=0, fixed_count=False):
    X = np.ascontiguousarray(X, np.float32)
    n, d = X.shape
    a = 1.0 / math.sqrt(d) if a is None else a
    mats, splits, offsets, indices = [], [], [], []
    for t in range(n_trees):
        R, (s, o, i) = build_one_tree(X, depth, a, seed, t, fixed_count)
        mats.append(R)
        splits.append(s)
        offsets.append(o)
        indices.append(i)
    return dict(matrices=mats, splits=np.stack(splits), leaf_offsets=np.stack(offsets),
                leaf_indices=np.stack(indices), depth=depth, n=n, d=d)


def query_leaves(Q, index):
    """Per-query leaf of every tree: _route_all (search.py:116-120)."""
    Q = np.ascontiguousarray(np.atleast_2d(Q), np.float32)
    T = len(index["matrices"])
    out = np.empty((Q.shape[0], T), dtype=np.int64)
    for t, R in enumerate(index["matrices"]):
        proj = project(Q, *R)
        out[:, t] = route(proj, np.repeat(index["splits"][t:t + 1], Q.shape[0], axis=0))
    return out


def vote_counts(leaves, index):
    n = index["leaf_indices"].shape[1]
    T = index["leaf_indices"].shape[0]
    counts = np.empty(n, dtype=np.int32)
    lib().oracle_vote_counts(np.ascontiguousarray(index["leaf_indices"], np.int32),
                             np.ascontiguousarray(index["leaf_offsets"], np.int64), n, T,
                             index["leaf_offsets"].shape[1] - 1,
                             np.ascontiguousarray(leaves, np.int64), counts)
    return counts


def candidates(leaves, index, v):
    """Sorted candidate set {id : votes >= v} (search.py:75-86, _py.vote)."""
    return np.flatnonzero(vote_counts(leaves, index) >= v).astype(np.int64)


def scan(X, cand, q):
    X = np.ascontiguousarray(X, np.float32)
    cand = np.ascontiguousarray(cand, np.int64)
    out = np.empty(cand.shape[0], dtype=np.float64)
    lib().oracle_scan(X, X.shape[1], cand, cand.shape[0], np.ascontiguousarray(q, np.float32), out)
    return out


def exact_knn(X, q, k, cand):
    """exact_knn_in_set (search.py:146-172): (ids i64, dists f64, candidate_count)."""
    S = np.unique(np.asarray(cand, dtype=np.int64).ravel())
    if S.shape[0] == 0:
        return np.zeros(0, np.int64), np.zeros(0, np.float64), 0
    d2 = scan(X, S, q)
    order = np.lexsort((S, d2))[:k]
    return S[order], np.sqrt(d2[order]), int(S.shape[0])


def approximate_knn_batch(X, Q, k, index, v):
    """approximate_knn (search.py:175-184) for every row of Q, padded like the
    product's batch API: ids -1 / dists +inf past min(k, |S|)."""
    Q = np.ascontiguousarray(np.atleast_2d(Q), np.float32)
    leaves = query_leaves(Q, index)
    nq = Q.shape[0]
    ids = np.full((nq, k), -1, dtype=np.int64)
    dists = np.full((nq, k), np.inf, dtype=np.float64)
    counts = np.zeros(nq, dtype=np.int64)
    for i in range(nq):
        S = candidates(leaves[i], index, v)
        a, b, c = exact_knn(X, Q[i], k, S)
        ids[i, :len(a)] = a
        dists[i, :len(b)] = b
        counts[i] = c
    return ids, dists, counts


def candidates_crossing_order(leaves, index, v):
    """The compiled reference's candidate order (_cy.pyx:57-78): trees in
    order, each leaf slice in stored order, an id emitted when its running
    count becomes exactly v."""
    L, O = index["leaf_indices"], index["leaf_offsets"]
    counts = {}
    out = []
    for t, leaf in enumerate(np.asarray(leaves, dtype=np.int64)):
        for idx in L[t, O[t, leaf]:O[t, leaf + 1]]:
            c = counts.get(int(idx), 0) + 1
            counts[int(idx)] = c
            if c == v:
                out.append(int(idx))
    return np.array(out, dtype=np.int64)


def pairwise_plan(n, lo=0):
    """numpy's pairwise summation of n contiguous float64 terms (numpy
    loops_utils.h pairwise_sum), as the postfix plan the GPU ground-truth
    kernel evaluates: ("leaf", lo, len) blocks of <= 128 terms and "add"."""
    if n <= 128:
        return [("leaf", lo, n)]
    n2 = n // 2
    n2 -= n2 % 8
    return pairwise_plan(n2, lo) + pairwise_plan(n - n2, lo + n2) + ["add"]


def pairwise_sum(a):
    """Restatement of numpy's pairwise float64 sum of a 1-D array: a leaf of
    < 8 terms is summed in order from 0.0; 8..128 terms go to 8 interleaved
    accumulators combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the n % 8
    tail in order; longer runs split at n/2 - (n/2) % 8."""
    a = [float(x) for x in a]
    stack = []
    for op in pairwise_plan(len(a)):
        if op == "add":
            r = stack.pop()
            stack.append(stack.pop() + r)
            continue
        _, lo, n = op
        if n < 8:
            res = 0.0
            for x in a[lo:lo + n]:
                res += x
        else:
            r = a[lo:lo + 8]
            m = n - n % 8
            for i in range(8, m, 8):
                for j in range(8):
                    r[j] += a[lo + i + j]
            res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
            for x in a[lo + m:lo + n]:
                res += x
        stack.append(res)
    return stack[0] if stack else 0.0


def brute_force_knn(X, q, k):
    """evaluation.brute_force_knn (evaluation.py:28-47): float64 differences,
    d2 = numpy's row sums (pairwise order, restated by pairwise_sum), the
    first min(k, n) of np.lexsort((ids, d2)); returns (ids, dists, n)."""
    X = np.ascontiguousarray(X, np.float32)
    qv = np.asarray(q, dtype=np.float64).ravel()
    diff = X.astype(np.float64) - qv
    d2 = (diff * diff).sum(axis=1)
    ids = np.arange(X.shape[0], dtype=np.int64)
    order = np.lexsort((ids, d2))[:k]
    return ids[order], np.sqrt(d2[order]), X.shape[0]


def compute_ground_truth(X, Q, k):
    """evaluation.compute_ground_truth (evaluation.py:65-81): (nq, k) ids and
    distances, one brute-force scan per query."""
    Q = np.atleast_2d(np.asarray(Q, dtype=np.float32))
    ids = np.empty((Q.shape[0], k), dtype=np.int64)
    dists = np.empty((Q.shape[0], k), dtype=np.float64)
    for i, q in enumerate(Q):
        a, b, _ = brute_force_knn(X, q, k)
        ids[i], dists[i] = a, b
    return ids, dists


def fnv1a64(buf):
    arr = np.ascontiguousarray(np.frombuffer(bytes(buf), dtype=np.uint8)
                               if isinstance(buf, (bytes, bytearray)) else
                               np.asarray(buf).view(np.uint8).reshape(-1))
    return int(lib().oracle_fnv1a64(arr, arr.shape[0]))
