"""Reference-side binding of libmrpt_cuda.so -- the module a maintainer of the
reference package would drop in next to its Cython backend, as
``pkg/src/mrpt/_kernels/_b200.py`` (the reference's plug-in point is
``mrpt._kernels``, _kernels/__init__.py:71-88; its compiled backend is
_kernels/_cy.pyx:18-106).

It binds the C ABI of include/mrpt_cuda.h with ctypes (argtypes below are
checked against the header by tests/test_abi.py) and offers the reference's
kernel calling conventions on host numpy arrays:

    project(data, col_ptr, rows, vals) -> f32[m, ncols]     (_cy.pyx:18-34)
    route(proj, splits)                -> i64[T]             (_cy.pyx:37-54)
    vote(leaf_indices, leaf_offsets, leaves, v, counts, stamps, epoch, out) -> ncand
                                                             (_cy.pyx:57-78)
    scan(data, cand, q)                -> f64[m] squared     (_cy.pyx:81-97)
    fnv1a64(buf)                       -> int                (_cy.pyx:100-106)

each computed on the GPU with results bit-identical to the Cython kernels
(vote returns the same candidate SET; its order is ascending, like the numpy
backend's _py.vote).  Per call it copies the operands to the device and the
result back, so through this per-tree / per-query interface the GPU pays a
launch and two copies per call; the batched entry points (mrpt_build_levels,
mrpt_query_route, mrpt_vote over a query matrix, mrpt_scan_topk) are where
the speed is, which is why paper_1509_06957_b200 exposes them at the API
level.  Device memory comes from PyTorch (buffers and the
current stream only).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_p, _i32, _i64, _sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t

# entry point -> argtypes (every function returns int32 status except the two below)
ARGTYPES = {
    "mrpt_last_error": [],
    "mrpt_project": [_p, _i64, _i32, _i64, _p, _p, _p, _i32, _p, _i64, _i64, _p],
    "mrpt_route": [_p, _i64, _i32, _p, _i64, _p, _p],
    "mrpt_vote_counts": [_p, _p, _i64, _i32, _i32, _p, _p, _p],
    "mrpt_select_ge": [_p, _i64, _i32, _p, _p, _p],
    "mrpt_scan": [_p, _i64, _i32, _i64, _p, _i64, _p, _p, _p],
    "mrpt_fnv1a64_workspace_size": [_i64, ctypes.POINTER(_sz)],
    "mrpt_fnv1a64": [_p, _i64, _p, _p, _sz, _p],
}
RESTYPES = {"mrpt_last_error": ctypes.c_char_p}

_lib = None


def _load(path=None):
    global _lib
    if _lib is None:
        path = path or os.environ.get("MRPT_CUDA_LIB", "libmrpt_cuda.so")
        lib = ctypes.CDLL(path)
        for name, args in ARGTYPES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = RESTYPES.get(name, ctypes.c_int32)
        _lib = lib
    return _lib


def _check(status):
    if status != 0:
        raise RuntimeError(_load().mrpt_last_error().decode())


def _dev(arr, dtype):
    import torch

    return torch.from_numpy(np.ascontiguousarray(arr, dtype=dtype)).cuda()


def _stream():
    import torch

    return torch.cuda.current_stream().cuda_stream


def project(data, col_ptr, rows, vals):
    """_cy.project: float32 (m, ncols), float64 sums in CSC order, rounded once."""
    import torch

    X = _dev(data, np.float32)
    cp, r, v = _dev(col_ptr, np.int64), _dev(rows, np.int32), _dev(vals, np.float32)
    ncols = len(col_ptr) - 1
    out = torch.empty((X.shape[0], ncols), dtype=torch.float32, device=X.device)
    _check(_load().mrpt_project(X.data_ptr(), X.shape[0], X.shape[1], X.shape[1], cp.data_ptr(),
                                r.data_ptr(), v.data_ptr(), ncols, out.data_ptr(), ncols, 1,
                                _stream()))
    return out.cpu().numpy()


def route(proj, splits):
    """_cy.route: leaf of every row (``p > split`` goes right)."""
    import torch

    P, S = _dev(proj, np.float32), _dev(splits, np.float32)
    out = torch.empty(P.shape[0], dtype=torch.int64, device=P.device)
    _check(_load().mrpt_route(P.data_ptr(), P.shape[0], P.shape[1], S.data_ptr(), S.shape[1],
                              out.data_ptr(), _stream()))
    return out.cpu().numpy()


def vote(leaf_indices, leaf_offsets, leaves, v, counts, stamps, epoch, out):
    """_cy.vote's contract: counts of the current epoch into ``counts``
    (``stamps`` set to ``epoch`` where touched), ids with count >= v into
    ``out``; returns their number."""
    import torch

    L, O = _dev(leaf_indices, np.int32), _dev(leaf_offsets, np.int64)
    T, n = L.shape
    depth = int(np.log2(O.shape[1] - 1))
    lv = _dev(np.asarray(leaves).astype(np.int32), np.int32)
    c = torch.empty(n, dtype=torch.int32, device=L.device)
    _check(_load().mrpt_vote_counts(L.data_ptr(), O.data_ptr(), n, T, depth, lv.data_ptr(),
                                    c.data_ptr(), _stream()))
    sel = torch.empty(n, dtype=torch.int32, device=L.device)
    ns = torch.zeros(1, dtype=torch.int64, device=L.device)
    _check(_load().mrpt_select_ge(c.data_ptr(), n, int(v), sel.data_ptr(), ns.data_ptr(),
                                  _stream()))
    ch = c.cpu().numpy()
    touched = ch > 0
    counts[touched] = ch[touched]
    stamps[touched] = epoch
    m = int(ns.item())
    out[:m] = sel[:m].cpu().numpy()
    return m


def scan(data, cand, q):
    """_cy.scan: squared float64 distances summed in coordinate order."""
    import torch

    X, c, qv = _dev(data, np.float32), _dev(cand, np.int64), _dev(q, np.float32)
    out = torch.empty(c.shape[0], dtype=torch.float64, device=X.device)
    _check(_load().mrpt_scan(X.data_ptr(), X.shape[0], X.shape[1], X.shape[1], c.data_ptr(),
                             c.shape[0], qv.data_ptr(), out.data_ptr(), _stream()))
    return out.cpu().numpy()


def fnv1a64(buf):
    """_cy.fnv1a64 over the raw bytes."""
    import torch

    b = _dev(np.frombuffer(bytes(buf), dtype=np.uint8) if isinstance(buf, (bytes, bytearray))
             else np.asarray(buf).view(np.uint8).reshape(-1), np.uint8)
    need = _sz(0)
    _check(_load().mrpt_fnv1a64_workspace_size(b.numel(), ctypes.byref(need)))
    ws = torch.empty(max(1, need.value), dtype=torch.uint8, device=b.device)
    out = torch.zeros(1, dtype=torch.int64, device=b.device)
    _check(_load().mrpt_fnv1a64(b.data_ptr(), b.numel(), out.data_ptr(), ws.data_ptr(),
                                need.value, _stream()))
    return int(out.item()) & 0xFFFFFFFFFFFFFFFF
