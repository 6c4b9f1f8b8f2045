"""The C-ABI library loads and exports every symbol declared in include/*.h
(no compute calls: runs on the CPU-only build container)."""
import ctypes
import glob
import os
import re

from paper_2602_12242_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(mxb_[a-z0-9_]+)\s*\(", src))
    return names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared()
    assert len(names) >= 30
    for n in sorted(names):
        assert hasattr(lib, n), n


def test_binding_covers_header():
    assert declared() == set(_lib.SIGNATURES)


def test_abi_version_and_error_string():
    lib = _lib.load()
    assert lib.mxb_abi_version() == 1
    assert isinstance(lib.mxb_last_error(), bytes)


def test_invalid_grid_rejected_without_gpu():
    lib = _lib.load()
    g = _lib.Grid(0, 1, 1, 1e-9, 1e-9, 1e-9)
    h = ctypes.c_void_p()
    assert lib.mxb_demag_create(ctypes.byref(g), 0, ctypes.byref(h)) == _lib.EINVAL
    assert b"cell counts" in lib.mxb_last_error()
