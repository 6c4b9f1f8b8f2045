"""The reference-side binding of INTEGRATION.md section 2, as a module.

This is the file a maintainer of the reference package would add as
``magnex/b200.py``: plain ctypes over the C-ABI of libmagnex_b200.so
(include/magnex_b200.h), no dependency on this repository's Python package.
``B200Demag`` plugs into the reference's demag seam
(``PartitionedRHS(demag=obj)``, obj.field(mdata) -> h, reference
llg.py:92-95,119-121) with a DemagKernel's packed tensor (demag.py:183-195).

tests/test_integration_binding.py runs it on the GPU through the same seam of
this package's PartitionedRHS.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_DEFAULT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "paper_2602_12242_b200", "libmagnex_b200.so")
_lib = ctypes.CDLL(os.environ.get("MAGNEX_B200_LIB", _DEFAULT))
_dp = ctypes.POINTER(ctypes.c_double)


class _Grid(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int64), ("ny", ctypes.c_int64), ("nz", ctypes.c_int64),
                ("dx", ctypes.c_double), ("dy", ctypes.c_double), ("dz", ctypes.c_double)]


for _name, _args in {"mxb_demag_create": [ctypes.POINTER(_Grid), ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)],
                     "mxb_demag_set_packed": [ctypes.c_void_p, _dp],
                     "mxb_demag_field": [ctypes.c_void_p, _dp, _dp],
                     "mxb_demag_destroy": [ctypes.c_void_p]}.items():
    getattr(_lib, _name).argtypes, getattr(_lib, _name).restype = _args, ctypes.c_int
_lib.mxb_last_error.restype = ctypes.c_char_p


def _check(rc):
    if rc:
        msg = _lib.mxb_last_error().decode()
        raise (ValueError if rc == 1 else RuntimeError)(msg)


class B200Demag:
    """DemagKernel-compatible backend: field(mdata) -> h (demag.py:203-216),
    evaluated on the GPU from the kernel's packed real-space tensor."""

    def __init__(self, kernel, device: int = 0):
        g = kernel.grid
        self.grid = g
        self.h = ctypes.c_void_p()
        _check(_lib.mxb_demag_create(ctypes.byref(_Grid(g.nx, g.ny, g.nz, g.dx, g.dy, g.dz)), device,
                                     ctypes.byref(self.h)))
        p = np.ascontiguousarray(kernel._packed, dtype=np.float64)
        _check(_lib.mxb_demag_set_packed(self.h, p.ctypes.data_as(_dp)))

    def field(self, mdata):
        m = np.ascontiguousarray(mdata, dtype=np.float64)
        g = self.grid
        if m.shape != (3, g.nz, g.ny, g.nx):
            raise ValueError(f"kernel built for {(g.nz, g.ny, g.nx)}, field is {m.shape[1:]}")
        h = np.empty_like(m)
        _check(_lib.mxb_demag_field(self.h, m.ctypes.data_as(_dp), h.ctypes.data_as(_dp)))
        return h

    def __del__(self):
        try:
            if self.h:
                _lib.mxb_demag_destroy(self.h)
        except Exception:
            pass
