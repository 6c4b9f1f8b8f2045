"""Demagnetising field by zero-padded FFT convolution (reference: demag.py).

``DemagKernel`` keeps the reference API (build / from_packed /
copy_workspace / field / spectra) but owns device-resident spectra and the
hand-written FFT pipeline of csrc/demag.cu.  ``DemagKernel.build`` runs the
Newell tensor builder on the GPU (csrc/newell.cu); ``from_packed`` accepts
the reference's exact packed real-space tensor (the parity path).
"""
from __future__ import annotations

import ctypes as C
import hashlib

import numpy as np

from . import _lib as L
from .grid import GridSpec, VectorField3

DIPOLE_SWITCH_DIAGONALS = 60.0   # demag.py:29
DIRECT_SUM_CELL_LIMIT = 4096     # demag.py:30
XX, XY, XZ, YY, YZ, ZZ = range(6)
_MIX = ((XX, XY, XZ), (XY, YY, YZ), (XZ, YZ, ZZ))


def _padded_dims(grid: GridSpec):
    """(pz, py, px): 2n per axis, 1 for a singleton axis (demag.py:152-155)."""
    return (2 * grid.nz if grid.nz > 1 else 1, 2 * grid.ny if grid.ny > 1 else 1,
            2 * grid.nx if grid.nx > 1 else 1)


class _Demag:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        try:
            if self.h:
                L.load().mxb_demag_destroy(self.h)
        except Exception:
            pass


class DemagKernel:
    """Device spectra plus FFT workspace for one grid (demag.py:169-216).

    Not reentrant (one evaluation at a time per instance), like the
    reference; ``copy_workspace`` gives an independent instance.
    """

    def __init__(self, grid: GridSpec, handle: _Demag, workers: int = 1, symmetric=False):
        self.grid = grid
        self.padded = _padded_dims(grid)
        self.workers = workers
        self._d = handle
        self.symmetric = symmetric

    @classmethod
    def _new(cls, grid: GridSpec) -> _Demag:
        lib = L.load()
        h = C.c_void_p()
        L.check(lib.mxb_demag_create(C.byref(grid._c()), L.device(), C.byref(h)), "demag_create")
        return _Demag(h)

    @classmethod
    def build(cls, grid: GridSpec, workers: int = 1, symmetric: bool = False) -> "DemagKernel":
        """GPU Newell tensor + spectra (demag.py:183-187).  ``symmetric=True``
        mirrors the displacement octant so the spectra are exactly real."""
        d = cls._new(grid)
        L.check(L.load().mxb_demag_build(d.h, 1 if symmetric else 0), "demag_build")
        return cls(grid, d, workers, symmetric)

    @classmethod
    def from_packed(cls, grid: GridSpec, packed: np.ndarray, workers: int = 1) -> "DemagKernel":
        """Spectra of a packed (6, pz, py, px) real-space tensor (demag.py:189-195)."""
        p = np.ascontiguousarray(packed, dtype=np.float64)
        if p.shape != (6,) + _padded_dims(grid):
            raise ValueError(f"packed kernel shape {p.shape} does not match {(6,) + _padded_dims(grid)}")
        d = cls._new(grid)
        L.check(L.load().mxb_demag_set_packed(d.h, L.dptr(p)), "demag_set_packed")
        k = cls(grid, d, workers)
        k._packed = p
        return k

    def copy_workspace(self) -> "DemagKernel":
        if hasattr(self, "_packed"):
            return DemagKernel.from_packed(self.grid, self._packed, self.workers)
        return DemagKernel.build(self.grid, self.workers, self.symmetric)

    @property
    def spectra(self) -> np.ndarray:
        """(6, pz, py, px//2+1) complex128, as scipy.fft.rfftn would return."""
        pz, py, px = self.padded
        out = np.empty((6, pz, py, px // 2 + 1, 2))
        L.check(L.load().mxb_demag_get_spectra(self._d.h, L.dptr(out)), "get_spectra")
        return out[..., 0] + 1j * out[..., 1]

    @property
    def pipeline(self) -> bool:
        """True when the y/z passes run as the L2-resident plane pipeline (yz_pipe.cu):
        kernel mode 3 (mirrored tensor, real quarter spectra) or 5 (any tensor,
        e.g. the reference's via ``from_packed``: full complex spectra)."""
        return self.kmode in (3, 5)

    @property
    def kmode(self) -> int:
        """Spectra storage: 0 complex (5-pass), 2 real quarter (5-pass), 3 real
        quarter (plane pipeline), 4 real quarter (long-y), 5 complex (plane pipeline)."""
        k = C.c_int()
        L.check(L.load().mxb_demag_kmode(self._d.h, C.byref(k)), "kmode")
        return k.value

    def set_fast(self, flag: bool) -> None:
        """Use the register-resident radix-16 kernels (default) or the generic
        mixed-radix kernels where both cover the shape."""
        L.check(L.load().mxb_demag_set_fast(self._d.h, 1 if flag else 0), "set_fast")

    @property
    def device_bytes(self) -> int:
        return int(L.load().mxb_demag_bytes(self._d.h))

    def field(self, mdata: np.ndarray) -> np.ndarray:
        """H_demag (A/m) of a (3, nz, ny, nx) magnetisation (demag.py:203-216)."""
        m = np.ascontiguousarray(mdata, dtype=np.float64)
        if m.shape != (3,) + self.grid.shape:
            raise ValueError(f"kernel built for {self.grid.shape}, field is {m.shape[1:]}")
        h = np.empty_like(m)
        L.check(L.load().mxb_demag_field(self._d.h, L.dptr(m), L.dptr(h)), "demag_field")
        return h


def demag_field_fft(m: VectorField3, kernel: DemagKernel) -> np.ndarray:
    """demag.py:219-222"""
    if m.grid.shape != kernel.grid.shape:
        raise ValueError(f"kernel built for {kernel.grid.shape}, field is {m.grid.shape}")
    return kernel.field(m.data)


def tensor_elements(nx: int, ny: int, nz: int, dx: float, dy: float, dz: float) -> np.ndarray:
    """(6, 2nz-1, 2ny-1, 2nx-1) cell-pair tensor from the GPU builder (demag.py:90-120)."""
    g = GridSpec(nx, ny, nz, dx, dy, dz)
    d = DemagKernel._new(g)
    out = np.empty((6, 2 * nz - 1, 2 * ny - 1, 2 * nx - 1))
    L.check(L.load().mxb_demag_tensor_elements(d.h, L.dptr(out)), "tensor_elements")
    return out


def self_demag_tensor(dx: float, dy: float, dz: float) -> np.ndarray:
    """3x3 self tensor of one cell (demag.py:144-149)."""
    n6 = tensor_elements(1, 1, 1, dx, dy, dz)[:, 0, 0, 0]
    return np.array([[n6[XX], n6[XY], n6[XZ]], [n6[XY], n6[YY], n6[YZ]],
                     [n6[XZ], n6[YZ], n6[ZZ]]])


def kernel_cache_name(grid: GridSpec) -> str:
    """demag.py:251-253"""
    key = f"{grid.nx},{grid.ny},{grid.nz},{grid.dx:.17g},{grid.dy:.17g},{grid.dz:.17g}"
    return "demag-" + hashlib.sha256(key.encode()).hexdigest()[:16] + ".magf"
