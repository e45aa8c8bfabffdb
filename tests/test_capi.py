"""The C-ABI library loads and exports every entry point include/mfh.h declares
(no compute calls — runs without a GPU)."""
import ctypes
import os
import re

from conftest import ROOT


def declared_functions():
    src = open(os.path.join(ROOT, "include", "mfh.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-zA-Z_][\w\s\*]*?\b(mfh_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("mfh_factorize", "mfh_apply", "mfh_gmres", "mfh_full_pivot_lu_batched",
                 "mfh_nd_create", "mfh_etree_create", "mfh_spmv", "mfh_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1410_2697_b200 import _lib
    L = _lib.lib()
    for name in declared_functions():
        assert hasattr(L, name), name
        assert isinstance(getattr(L, name), ctypes._CFuncPtr)
    # the python binding covers the whole header
    assert set(declared_functions()) <= set(_lib.EXPORTED)


def test_error_translation_without_gpu():
    import numpy as np
    import pytest
    from paper_1410_2697_b200 import _lib
    with pytest.raises(ValueError, match="leaf_size"):
        h = ctypes.c_void_p()
        ip = np.zeros(2, dtype=np.int64)
        _lib.check(_lib.lib().mfh_nd_create(1, _lib.ptr(ip), _lib.ptr(ip), 0, ctypes.byref(h)))
