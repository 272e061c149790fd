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


# --- argument lists: every binding's argtypes against the header ---------------
_CT = {"int32_t": ctypes.c_int32, "int64_t": ctypes.c_int64, "size_t": ctypes.c_size_t,
       "double": ctypes.c_double, "uint64_t": ctypes.c_uint64}


def header_argtypes():
    """name -> ctypes argtypes implied by include/mrpt_cuda.h: scalars by type,
    pointers annotated /* host */ as POINTER(base), every other pointer (device
    memory, streams, events) as c_void_p."""
    text = open(HEADER).read().replace("/* host */", " __HOST__ ")
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    out = {}
    for m in re.finditer(r"\b(?:int32_t|int64_t|const char \*)\s*(mrpt_[a-z0-9_]+)\s*\((.*?)\)\s*;",
                         text, flags=re.S):
        name, params = m.group(1), m.group(2)
        params = re.sub(r"\s+", " ", params).strip()
        args = []
        if params and params != "void":
            for prm in params.split(","):
                host = "__HOST__" in prm
                prm = prm.replace("__HOST__", "").replace("const ", "").strip()
                if "*" in prm:
                    base = prm.split("*")[0].strip()
                    args.append(ctypes.POINTER(_CT[base]) if host else ctypes.c_void_p)
                else:
                    args.append(_CT[prm.rsplit(" ", 1)[0].strip()])
        out[name] = args
    return out


def test_native_argtypes_match_header():
    hdr = header_argtypes()
    for name, args in _native.SIGNATURES.items():
        assert args == hdr[name], name


def test_reference_side_binding_matches_header():
    """bindings/_b200.py (the ctypes module a reference maintainer would add)
    and bindings/mrpt_cuda.pxd (the Cython declarations) agree with the
    header parameter for parameter."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("_b200", os.path.join(ROOT, "bindings", "_b200.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    hdr = header_argtypes()
    for name, args in mod.ARGTYPES.items():
        assert args == hdr[name], name
    pxd = open(os.path.join(ROOT, "bindings", "mrpt_cuda.pxd")).read()
    text = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    norm = lambda s: [re.sub(r"\s+", " ", p.replace("const ", "")).strip().rsplit(" ", 1)[0].replace(" *", "*")
                      for p in s.split(",") if p.strip() and p.strip() != "void"]
    for m in re.finditer(r"(mrpt_[a-z0-9_]+)\((.*?)\)", pxd, flags=re.S):
        h = re.search(m.group(1) + r"\s*\((.*?)\)\s*;", text, flags=re.S)
        assert h, m.group(1)
        assert [t.replace("*", "").strip() for t in norm(m.group(2))] == \
            [t.replace("*", "").strip() for t in norm(h.group(1))], m.group(1)
