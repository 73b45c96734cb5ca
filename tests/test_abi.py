"""The C-ABI library loads without a GPU and exports every symbol that
include/plv.h declares (no compute calls here)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT

from paper_1410_1237_b200 import _lib

HEADER = os.path.join(ROOT, "include", "plv.h")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(plv_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("plv_csr_build", "plv_decide", "plv_apply", "plv_color", "plv_vf_records",
                 "plv_rebuild_records", "plv_modularity", "plv_phase_create", "plv_phase_run"):
        assert must in names


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libplv.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    assert set(declared()) == set(_lib.exported_symbols())


def test_no_device_means_explicit_failure():
    """Without an sm_100 device the library reports it instead of computing
    anything on the CPU (there is no fallback)."""
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libplv.so not built")
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    L = _lib.lib()
    assert L.device_ok() == 0
    out = ctypes.c_double()
    rc = L.sum(None, 0, ctypes.addressof(out), None)
    assert rc == _lib.PLV_ENODEV
    assert b"no CUDA device" in L.last_error() or b"sm_100" in L.last_error()
