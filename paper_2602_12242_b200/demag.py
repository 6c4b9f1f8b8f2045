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
from . import io as mio
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
        k = cls(grid, d, workers, symmetric)
        k._built = True
        return k

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

    def __getattr__(self, name):
        # the packed real-space tensor of a GPU-built kernel (reference
        # DemagKernel.build keeps it via from_packed, demag.py:183-195), formed
        # on first use from the GPU builder's elements and the wrap-around pack
        if name == "_packed" and "_d" in self.__dict__:
            g = self.grid
            n6 = tensor_elements(g.nx, g.ny, g.nz, g.dx, g.dy, g.dz)
            if self.symmetric:
                n6 = _mirror(n6)
            self.__dict__["_packed"] = _pack_wraparound(n6, g)
            return self.__dict__["_packed"]
        raise AttributeError(name)

    def copy_workspace(self) -> "DemagKernel":
        if "_packed" in self.__dict__ and not getattr(self, "_built", False):
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


def demag_field_direct(m: VectorField3, grid: GridSpec, n6: np.ndarray | None = None) -> np.ndarray:
    """O(N^2) direct sum over source cells on the GPU (demag.py:225-248): the
    oracle of the FFT path, limited to DIRECT_SUM_CELL_LIMIT cells.  ``n6``
    (6, 2nz-1, 2ny-1, 2nx-1) supplies the tensor elements; by default the GPU
    builder's (the reference recomputes tensor_elements here too)."""
    if grid.n_cells > DIRECT_SUM_CELL_LIMIT:
        raise ValueError(
            f"direct sum limited to {DIRECT_SUM_CELL_LIMIT} cells, grid has {grid.n_cells}")
    md = np.ascontiguousarray(m.data, dtype=np.float64)
    if md.shape != (3,) + grid.shape:
        raise ValueError(f"field has shape {md.shape[1:]}, grid is {grid.shape}")
    nx, ny, nz = grid.nx, grid.ny, grid.nz
    e = None
    if n6 is not None:
        e = np.ascontiguousarray(n6, dtype=np.float64)
        if e.shape != (6, 2 * nz - 1, 2 * ny - 1, 2 * nx - 1):
            raise ValueError(f"tensor elements have shape {e.shape}")
    d = DemagKernel._new(grid)
    h = np.empty_like(md)
    L.check(L.load().mxb_demag_direct(d.h, L.dptr(e) if e is not None else None, L.dptr(md), L.dptr(h)),
            "demag_direct")
    return h


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


# (x, y, z) parity of XX, XY, XZ, YY, YZ, ZZ under a sign flip of that axis
_PARITY = ((1, 1, 1), (-1, -1, 1), (-1, 1, -1), (1, 1, 1), (1, -1, -1), (1, 1, 1))


def _mirror(n6: np.ndarray) -> np.ndarray:
    """The non-negative displacement octant mirrored with the exact parities
    (what build(symmetric=True) evaluates on the GPU)."""
    out = np.empty_like(n6)
    _, Z, Y, X = n6.shape
    idx = [np.abs(np.arange(n) - n // 2) + n // 2 for n in (Z, Y, X)]
    neg = [np.where(np.arange(n) < n // 2, -1.0, 1.0) for n in (Z, Y, X)]
    for c in range(6):
        px, py, pz = _PARITY[c]
        sign = np.ones((Z, Y, X))
        if pz < 0:
            sign *= neg[0][:, None, None]
        if py < 0:
            sign *= neg[1][None, :, None]
        if px < 0:
            sign *= neg[2][None, None, :]
        out[c] = sign * n6[c][np.ix_(*idx)]
    return out


def _pack_wraparound(n6: np.ndarray, grid: GridSpec) -> np.ndarray:
    """Displacement d -> padded index d mod p (demag.py:158-166)."""
    pz, py, px = _padded_dims(grid)
    packed = np.zeros((6, pz, py, px))
    iz = np.arange(-(grid.nz - 1), grid.nz) % pz
    iy = np.arange(-(grid.ny - 1), grid.ny) % py
    ix = np.arange(-(grid.nx - 1), grid.nx) % px
    packed[np.ix_(range(6), iz, iy, ix)] = n6
    return packed


def save_kernel(path, kernel: DemagKernel) -> None:
    """Write the packed real-space kernel as a 6-component MAGF file on the
    padded grid with the original cell sizes (demag.py:256-268)."""
    g = kernel.grid
    pz, py, px = kernel.padded
    mio.write_magf(path, kernel._packed, GridSpec(px, py, pz, g.dx, g.dy, g.dz))


def load_kernel(path, grid: GridSpec, workers: int = 1) -> DemagKernel:
    """Kernel from a save_kernel file, validated against the grid (demag.py:271-277)."""
    pgrid, packed = mio.read_magf(path)
    if packed.shape[0] != 6:
        raise mio.MagfError(f"{path}: kernel cache must hold 6 components")
    if (pgrid.nx, pgrid.ny, pgrid.nz) != _padded_dims(grid)[::-1] or \
            (pgrid.dx, pgrid.dy, pgrid.dz) != (grid.dx, grid.dy, grid.dz):
        raise mio.MagfError(f"{path}: cached kernel does not match the requested grid")
    return DemagKernel.from_packed(grid, packed, workers)


def kernel_cache_name(grid: GridSpec) -> str:
    """demag.py:251-253"""
    key = f"{grid.nx},{grid.ny},{grid.nz},{grid.dx:.17g},{grid.dy:.17g},{grid.dz:.17g}"
    return "demag-" + hashlib.sha256(key.encode()).hexdigest()[:16] + ".magf"
