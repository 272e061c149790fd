"""The C ABI: libmrpt_cuda.so loads without a GPU and exports exactly what
include/mrpt_cuda.h declares; host-side validation fails fast with the
documented status codes (no device work is enqueued)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT
from paper_1509_06957_b200 import _native

HEADER = os.path.join(ROOT, "include", "mrpt_cuda.h")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mrpt_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_native.LIB_PATH):
        import __graft_entry__

        __graft_entry__.build_native()
    return _native.load()


def test_header_and_binding_agree():
    assert declared() == sorted(_native.SIGNATURES)


def test_every_declared_symbol_is_exported(lib):
    for name in declared():
        assert hasattr(lib, name), name


def test_version_and_error_text(lib):
    assert lib.mrpt_abi_version() == 101
    assert lib.mrpt_launch_count() == 0  # nothing launched in this CPU-only process
    sz = ctypes.c_size_t(0)
    st = lib.mrpt_build_workspace_size(0, 1, 3, ctypes.byref(sz))
    assert st == _native.MRPT_ESHAPE
    assert b"n must lie" in lib.mrpt_last_error()
    st = lib.mrpt_build_workspace_size(1000, 0, 3, ctypes.byref(sz))
    assert st == _native.MRPT_EPARAM
    st = lib.mrpt_build_workspace_size(1000, 4, 5, ctypes.byref(sz))
    assert st == _native.MRPT_OK and sz.value > 4 * 1000 * 4


def test_status_maps_to_reference_exceptions(lib):
    from paper_1509_06957_b200 import ParameterError, ShapeError

    sz = ctypes.c_size_t(0)
    with pytest.raises(ShapeError):
        _native.call("mrpt_build_workspace_size", 0, 1, 3, ctypes.byref(sz))
    with pytest.raises(ParameterError):
        _native.call("mrpt_build_workspace_size", 10, 1, 40, ctypes.byref(sz))
    # vote: threshold above the possible count is rejected before any launch
    with pytest.raises(ParameterError):
        _native.call("mrpt_vote", None, None, 100, 4, 3, None, 1, 5, 1, 4, None, None, 10, None,
                     None)
    with pytest.raises(ParameterError):
        _native.call("mrpt_scan_topk", None, 10, 4, 4, None, 1, 4, None, 0, None, 0, None, None,
                     None)
