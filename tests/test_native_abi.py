"""The C-ABI library loads (no GPU needed) and exports every entry point that
include/amrb.h declares; the ctypes binding covers all of them (CPU)."""

import os
import re

import pytest

from paper_2009_12009_b200 import _native

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "amrb.h")


def _declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(amrb_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    names = _declared()
    assert len(names) > 20
    for n in names:
        assert hasattr(lib, n), n


def test_binding_covers_header():
    assert sorted(_native.EXPORTED) == _declared()


def test_error_mapping_without_gpu():
    import ctypes as C

    lib = _native.lib()
    h = C.c_void_p()
    st = lib.amrb_plan_fill_create(4, 0, None, 1, None, None, C.byref(h))
    assert st == _native.AMRB_EINVAL
    with pytest.raises(ValueError):
        _native.check(st)
    assert b"bad arguments" in lib.amrb_last_error()
