"""The C-ABI library builds, loads and exports every symbol include/*.h declares (CPU only)."""

import glob
import os
import re

from paper_2311_17500_b200 import _lib
from paper_2311_17500_b200.build import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        txt = open(h).read()
        names |= set(re.findall(r"^\s*(?:int|const char\*)\s+(mi_\w+)\s*\(", txt, re.M))
    return names


def test_library_exports_every_declared_symbol():
    build()
    lib = _lib.load()
    names = declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert names == set(_lib.EXPORTED)
    assert lib.mi_version() == 1


def test_no_device_needed_for_error_path():
    lib = _lib.load()
    import ctypes
    h = ctypes.c_void_p()
    import numpy as np
    dims = np.array([4], dtype=np.int32)
    rc = lib.mi_ctx_create(0, 5, ctypes.c_void_p(dims.ctypes.data), 4, 2, 2, ctypes.byref(h))
    assert rc == _lib.MI_ERR_ARG
    assert b"d must be" in lib.mi_last_error()
