"""The C ABI library loads (no GPU needed to dlopen) and exports every
function include/accfem.h declares; the ctypes layout matches the header."""

import ctypes
import os
import re

import pytest

from paper_2503_06922_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "accfem.h")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(accfem_[a-z_]+)\s*\(", text)))


def test_header_declares_the_binding():
    assert set(declared()) == set(_lib.SIGNATURES)


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.fail("libaccfem.so not built: run __graft_entry__.build()")
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared():
        assert hasattr(lib, name), name
    _lib.bind(lib)
    assert lib.accfem_version() == 1


def test_batch_struct_field_order_matches_header():
    text = open(HEADER).read()
    body = text[text.index("typedef struct {\n  int32_t S;"):text.index("} accfem_batch;")]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    names = re.findall(r"\b([A-Za-z_0-9]+);", body)
    assert names == [f for f, _ in _lib.BATCH_FIELDS]


def test_create_without_gpu_reports_error_not_crash():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2503_06922_b200 import DeviceError, scenarios
    from paper_2503_06922_b200.engine import Engine
    w = scenarios.cfg3p(1)
    with pytest.raises(DeviceError):
        Engine(**w.engine_kwargs())
