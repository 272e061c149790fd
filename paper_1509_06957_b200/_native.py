"""ctypes binding of libmrpt_cuda.so (the C ABI declared in include/mrpt_cuda.h).

This is the only way the package reaches the device: there is no CPU or
Python fallback.  If the library is missing or no CUDA device is present,
every compute entry point raises :class:`DeviceError` immediately.
Tensors cross the boundary as raw device pointers (``tensor.data_ptr()``)
and the work is enqueued on the caller's current torch CUDA stream.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .exceptions import DeviceError, IntegrityError, MRPTError, ParameterError, ShapeError

LIB_NAME = "libmrpt_cuda.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

_c_i32, _c_i64, _c_p, _c_sz = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t

# name -> argtypes; every function returns int32 status unless listed in _RESTYPE
SIGNATURES = {
    "mrpt_last_error": [],
    "mrpt_abi_version": [],
    "mrpt_launch_count": [],
    "mrpt_project": [_c_p, _c_i64, _c_i32, _c_i64, _c_p, _c_p, _c_p, _c_i32, _c_p, _c_i64, _c_i64, _c_p],
    "mrpt_route": [_c_p, _c_i64, _c_i32, _c_p, _c_i64, _c_p, _c_p],
    "mrpt_query_route": [_c_p, _c_i64, _c_i32, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_i32, _c_i32, _c_p,
                         _c_p],
    "mrpt_build_workspace_size": [_c_i64, _c_i32, _c_i32, ctypes.POINTER(_c_sz)],
    "mrpt_build_levels": [_c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_p, _c_p, _c_sz, _c_p],
    "mrpt_vote": [_c_p, _c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_i64, _c_i32, _c_i32, _c_i64, _c_p,
                  _c_p, _c_i64, _c_p, _c_p],
    "mrpt_vote_plan": [_c_i64, _c_i32, _c_i32, _c_i64, ctypes.POINTER(_c_i32), ctypes.POINTER(_c_i64)],
    "mrpt_vote_build_dir": [_c_p, _c_p, _c_i64, _c_i32, _c_i32, _c_i64, _c_p, _c_p],
    "mrpt_vote_stream_plan": [_c_i64, _c_i32, _c_i32, _c_i64, ctypes.POINTER(_c_i32),
                              ctypes.POINTER(_c_i64)],
    "mrpt_vote_stream_layout": [_c_p, _c_p, _c_i64, _c_i32, _c_i32, _c_i64, _c_p, _c_p, _c_p, _c_p],
    "mrpt_vote_stream_fill": [_c_p, _c_p, _c_i64, _c_i32, _c_i32, _c_i64, _c_p, _c_p, _c_i64, _c_p,
                              _c_p],
    "mrpt_vote_stream": [_c_p, _c_i64, _c_p, _c_p, _c_i64, _c_i32, _c_i32, _c_i64, _c_p, _c_i64,
                         _c_i32, _c_p, _c_i64, _c_p, _c_p],
    "mrpt_vote_pair_max_votes": [_c_i64, _c_i32, _c_i64, ctypes.POINTER(_c_i32)],
    "mrpt_vote_stats": [ctypes.POINTER(_c_i64), _c_i32],
    "mrpt_vote_pair_plan": [_c_i64, _c_i32, _c_i32, _c_i64, ctypes.POINTER(_c_i32),
                            ctypes.POINTER(_c_i64), ctypes.POINTER(_c_i64)],
    "mrpt_vote_pair_layout": [_c_p, _c_p, _c_i64, _c_i32, _c_i32, _c_i64, _c_p, _c_p, _c_p, _c_p,
                              _c_p],
    "mrpt_vote_pair_fill": [_c_p, _c_p, _c_i64, _c_i32, _c_i32, _c_i64, _c_p, _c_p, _c_p, _c_i64,
                            _c_p, _c_p],
    "mrpt_vote_pair": [_c_p, _c_i64, _c_p, _c_p, _c_i64, _c_i32, _c_i32, _c_i64, _c_p, _c_i64,
                       _c_i32, _c_p, _c_i64, _c_p, _c_p],
    "mrpt_vote_counts": [_c_p, _c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_p],
    "mrpt_select_ge": [_c_p, _c_i64, _c_i32, _c_p, _c_p, _c_p],
    "mrpt_scan": [_c_p, _c_i64, _c_i32, _c_i64, _c_p, _c_i64, _c_p, _c_p, _c_p],
    "mrpt_scan_topk": [_c_p, _c_i64, _c_i32, _c_i64, _c_p, _c_i64, _c_i64, _c_p, _c_i64, _c_p,
                       _c_i32, _c_p, _c_p, _c_p],
    "mrpt_quantize_fp16": [_c_p, _c_i64, _c_i32, _c_i64, _c_p, _c_i64, _c_p, _c_p, _c_p],
    "mrpt_scan_topk_fp16": [_c_p, _c_i64, _c_i32, _c_i64, _c_p, _c_i64, _c_p, _c_p, _c_i64, _c_i64,
                            _c_p, _c_i64, _c_p, _c_i32, _c_p, _c_p, _c_p],
    "mrpt_quantize_u8": [_c_p, _c_i64, _c_i32, _c_i64, _c_p, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p],
    "mrpt_scan_topk_u8": [_c_p, _c_i64, _c_i32, _c_i64, _c_p, _c_i64, _c_p, _c_p, _c_p, _c_p,
                          _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_i32, _c_p, _c_p, _c_p],
    "mrpt_u8_gemm_rows": [_c_p, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p],
    "mrpt_vote_counted": [_c_p, _c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_i64, _c_i32, _c_i32, _c_i64,
                          _c_p, _c_p, _c_p, _c_i64, _c_p, _c_p],
    "mrpt_filter_counts": [_c_p, _c_p, _c_i64, _c_p, _c_i64, _c_i32, _c_p, _c_i64, _c_p, _c_p],
    "mrpt_vote_bitmap": [_c_p, _c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_i64, _c_i32, _c_i32, _c_i64,
                         _c_p, _c_p, _c_i64, _c_p, _c_p],
    "mrpt_scan_topk_u8tc_workspace_size": [_c_i64, _c_i64, _c_i64, ctypes.POINTER(_c_i64)],
    "mrpt_scan_topk_u8tc_bits": [_c_p, _c_i64, _c_i32, _c_i64, _c_p, _c_i64, _c_p, _c_p, _c_i64,
                                 _c_i64, _c_p, _c_i64, _c_i32, _c_p, _c_p, _c_p, _c_i64, _c_p, _c_p],
    "mrpt_kernel_timer": [_c_i32],
    "mrpt_fallback_stats": [ctypes.POINTER(_c_i64), _c_i32],
    "mrpt_kernel_timer_read": [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_c_i64)],
    "mrpt_unique_ids": [_c_p, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p],
    "mrpt_fnv1a64_workspace_size": [_c_i64, ctypes.POINTER(_c_sz)],
    "mrpt_fnv1a64": [_c_p, _c_i64, _c_p, _c_p, _c_sz, _c_p],
    "mrpt_brute_force_workspace_size": [_c_i64, _c_i32, _c_i64, _c_i32, ctypes.POINTER(_c_i64)],
    "mrpt_brute_force_knn": [_c_p, _c_i64, _c_i32, _c_i64, _c_p, _c_i64, _c_i64, _c_i32, _c_p, _c_p,
                             _c_p, _c_i64, _c_p],
    "mrpt_query_order": [_c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_p],
    "mrpt_permute_rows": [_c_p, _c_i64, _c_p, _c_i64, _c_i64, _c_p, _c_i64, _c_i32, _c_p],
    "mrpt_check_finite": [_c_p, _c_i64, _c_p, _c_p],
    "mrpt_audit_leaves": [_c_p, _c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p],
}
_RESTYPE = {"mrpt_last_error": ctypes.c_char_p, "mrpt_launch_count": _c_i64}

MRPT_OK, MRPT_EPARAM, MRPT_ESHAPE, MRPT_EINTEGRITY, MRPT_EWORKSPACE = 0, -1, -2, -3, -4
MRPT_ECUDA, MRPT_ENCCL = -10, -11

_lock = threading.Lock()
_lib = None


def load():
    """Load the shared library (no GPU needed to load it); raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise DeviceError(
                    f"{LIB_NAME} not built at {LIB_PATH}; run `python -c 'import __graft_entry__ as g; "
                    "g.build()'` (there is no CPU fallback)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, argtypes in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = argtypes
                fn.restype = _RESTYPE.get(name, _c_i32)
            _lib = lib
    return _lib


def check(status, what=""):
    if status == MRPT_OK:
        return
    msg = load().mrpt_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if status == MRPT_EPARAM:
        raise ParameterError(text)
    if status == MRPT_ESHAPE:
        raise ShapeError(text)
    if status == MRPT_EINTEGRITY:
        raise IntegrityError(text)
    if status in (MRPT_ECUDA, MRPT_ENCCL):
        raise DeviceError(text)
    raise MRPTError(f"status {status}: {text}")


def call(name, *args):
    """Invoke a C-ABI entry point and map its status onto the exception taxonomy."""
    check(getattr(load(), name)(*args), name)


def require_device():
    """The torch module, after checking a CUDA device and the library exist."""
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("a CUDA device is required: this package runs the MRPT hot path "
                          "only on the GPU (no CPU fallback)")
    load()
    return torch


def stream_ptr():
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    """Device pointer of a torch tensor (None -> NULL)."""
    return ctypes.c_void_p(0 if t is None else t.data_ptr())
