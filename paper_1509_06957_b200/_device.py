"""Device buffers and host<->device plumbing (torch is only the carrier)."""

from __future__ import annotations

import numpy as np

from . import _native


def torch_mod():
    return _native.require_device()


def device():
    torch = torch_mod()
    return torch.device("cuda", torch.cuda.current_device())


_SMS = {}


def sm_count():
    """Streaming multiprocessors of the current device."""
    torch = torch_mod()
    dev = torch.cuda.current_device()
    if dev not in _SMS:
        _SMS[dev] = int(torch.cuda.get_device_properties(dev).multi_processor_count)
    return _SMS[dev]


def is_tensor(x):
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


_SIDE = {}


def side_streams():
    """Two CUDA streams per device (upload, download) for overlapped batches."""
    torch = torch_mod()
    dev = torch.cuda.current_device()
    if dev not in _SIDE:
        _SIDE[dev] = (torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev))
    return _SIDE[dev]


_VOTE = {}


def vote_stream():
    """A CUDA stream per device for K3 running beside K4's GEMM."""
    torch = torch_mod()
    dev = torch.cuda.current_device()
    if dev not in _VOTE:
        _VOTE[dev] = torch.cuda.Stream(device=dev)
    return _VOTE[dev]


def h2d(arr, dtype=None):
    """Copy a host array to the current device (pinned staging for big arrays)."""
    torch = torch_mod()
    a = np.ascontiguousarray(arr if dtype is None else np.asarray(arr, dtype=dtype))
    if not a.flags.writeable:  # torch wants writable storage; the copy is read-only to us
        a = a.copy()
    t = torch.from_numpy(a)
    if a.nbytes >= (1 << 20):
        t = t.pin_memory()
        return t.to(device(), non_blocking=True)
    return t.to(device())


def d2h(t):
    return t.detach().cpu().numpy()


def empty(shape, dtype):
    torch = torch_mod()
    return torch.empty(shape, dtype=dtype, device=device())


def concat_csc(matrices):
    """Host CSC arrays of several SparseProjectionMatrix concatenated column-wise
    with global offsets (tree t owns columns t*depth .. t*depth+depth-1)."""
    ptrs, rows, vals = [np.zeros(1, np.int64)], [], []
    base = 0
    for R in matrices:
        cp = np.asarray(R.col_ptr, dtype=np.int64)
        ptrs.append(cp[1:] + base)
        rows.append(np.asarray(R.row_idx, dtype=np.int32))
        vals.append(np.asarray(R.values, dtype=np.float32))
        base += int(cp[-1])
    col_ptr = np.concatenate(ptrs)
    row_idx = np.concatenate(rows) if base else np.zeros(1, np.int32)
    values = np.concatenate(vals) if base else np.zeros(1, np.float32)
    return col_ptr, row_idx, values


def csc_device(matrices, pinned=False):
    """Device copies of the concatenated CSC arrays.  ``pinned`` stages them in
    page-locked memory and copies asynchronously, so the host can go on
    sampling the next batch while the stream is still busy."""
    cp, r, v = concat_csc(matrices)
    if not pinned:
        return h2d(cp), h2d(r), h2d(v)
    torch = torch_mod()
    out = []
    for a in (cp, r, v):
        t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        out.append(t.to(device(), non_blocking=True))
    return tuple(out)
