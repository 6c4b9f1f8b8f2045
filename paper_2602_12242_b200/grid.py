"""Grid, field and material containers (reference: grid.py).

Host-side containers keep the reference layout: float64 (3, nz, ny, nx),
C-contiguous, x fastest (grid.py:1-8).  A MaterialMap lazily owns one device
context (``mxb_ctx``) holding its parameters in HBM; every operator on that
material (renormalize, mean, the field terms, the stepping loop) runs through
that context on the GPU.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib as L

MU0 = 4.0e-7 * math.pi  # grid.py:17
GAMMA = -1.759e11  # grid.py:18


class GridError(ValueError):
    """grid.py:21"""


class RenormalizeError(ValueError):
    """Raised when a magnetic cell holds a zero vector (grid.py:25-26)."""


@dataclass(frozen=True)
class GridSpec:
    """Regular grid geometry (grid.py:29-71)."""

    nx: int
    ny: int
    nz: int
    dx: float
    dy: float
    dz: float
    origin: tuple = (0.0, 0.0, 0.0)

    def __post_init__(self):
        if min(self.nx, self.ny, self.nz) < 1:
            raise GridError(f"cell counts must be >= 1, got {(self.nx, self.ny, self.nz)}")
        if min(self.dx, self.dy, self.dz) <= 0.0:
            raise GridError(f"cell sizes must be > 0, got {(self.dx, self.dy, self.dz)}")

    @property
    def shape(self):
        return (self.nz, self.ny, self.nx)

    @property
    def n_cells(self) -> int:
        return self.nx * self.ny * self.nz

    @property
    def cell_volume(self) -> float:
        return self.dx * self.dy * self.dz

    @property
    def extent(self):
        return (self.nx * self.dx, self.ny * self.dy, self.nz * self.dz)

    def cell_centers(self):
        ox, oy, oz = self.origin
        xs = ox + (np.arange(self.nx) + 0.5) * self.dx
        ys = oy + (np.arange(self.ny) + 0.5) * self.dy
        zs = oz + (np.arange(self.nz) + 0.5) * self.dz
        Z, Y, X = np.meshgrid(zs, ys, xs, indexing="ij")
        return X, Y, Z

    def _c(self) -> L.Grid:
        return L.Grid(self.nx, self.ny, self.nz, self.dx, self.dy, self.dz)


class VectorField3:
    """3-component cell field, ``data`` shape (3, nz, ny, nx) float64 (grid.py:74-107)."""

    __slots__ = ("grid", "data")

    def __init__(self, grid: GridSpec, data: np.ndarray | None = None):
        self.grid = grid
        if data is None:
            data = np.zeros((3,) + grid.shape)
        else:
            data = np.ascontiguousarray(data, dtype=np.float64)
            if data.shape != (3,) + grid.shape:
                raise GridError(f"field shape {data.shape} does not match grid {(3,) + grid.shape}")
        self.data = data

    @classmethod
    def zeros(cls, grid: GridSpec) -> "VectorField3":
        return cls(grid)

    @classmethod
    def from_uniform(cls, grid: GridSpec, vec) -> "VectorField3":
        f = cls(grid)
        for c in range(3):
            f.data[c] = vec[c]
        return f

    def copy(self) -> "VectorField3":
        return VectorField3(self.grid, self.data.copy())

    def norm(self) -> np.ndarray:
        d = self.data
        return np.sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2])


def _cell_param(value, shape, name):
    arr = np.asarray(value, dtype=np.float64)
    if arr.ndim == 0:
        return np.full(shape, float(arr)), float(arr)
    if arr.shape != shape:
        raise GridError(f"{name} has shape {arr.shape}, expected scalar or {shape}")
    arr = np.ascontiguousarray(arr)
    if arr.size and np.all(arr == arr.flat[0]):
        return arr, float(arr.flat[0])
    return arr, None


class MaterialMap:
    """Per-cell Ms, A, Ku, D, alpha, eK plus gamma (grid.py:119-175).

    Extensions with no reference counterpart (parity unpinned): cubic
    anisotropy ``Kc1`` with axes ``c1``, ``c2`` and bulk DMI ``Db``.
    """

    def __init__(self, grid: GridSpec, Ms, A=0.0, Ku=0.0, eK=(0.0, 0.0, 1.0), D=0.0,
                 alpha=0.0, gamma: float = GAMMA, *, Kc1: float = 0.0, c1=(1.0, 0.0, 0.0),
                 c2=(0.0, 1.0, 0.0), Db: float = 0.0):
        shape = grid.shape
        self.grid = grid
        self.Ms, self._Ms_u = _cell_param(Ms, shape, "Ms")
        self.A, self._A_u = _cell_param(A, shape, "A")
        self.Ku, self._Ku_u = _cell_param(Ku, shape, "Ku")
        self.D, self._D_u = _cell_param(D, shape, "D")
        self.alpha, self._alpha_u = _cell_param(alpha, shape, "alpha")
        self.gamma = float(gamma)
        e = np.asarray(eK, dtype=np.float64)
        if e.shape == (3,):
            ek = np.empty((3,) + shape)
            for c in range(3):
                ek[c] = e[c]
        elif e.shape == (3,) + shape:
            ek = np.ascontiguousarray(e)
        else:
            raise GridError(f"eK has shape {e.shape}, expected (3,) or {(3,) + shape}")
        n = np.sqrt(np.einsum("cijk,cijk->ijk", ek, ek))
        if np.any((n == 0.0) & (self.Ku != 0.0)):
            raise GridError("eK must be nonzero wherever Ku != 0")
        with np.errstate(invalid="ignore", divide="ignore"):
            ek = np.where(n > 0.0, ek / n, 0.0)
        self.eK = ek
        flat = ek.reshape(3, -1)
        self._eK_u = tuple(float(v) for v in flat[:, 0]) if (
            flat.shape[1] and np.all(flat == flat[:, :1])) else None
        if np.any(self.Ms < 0.0):
            raise GridError("Ms must be >= 0")
        if np.any((self.D != 0.0) & (self.A <= 0.0) & (self.Ms > 0.0)):
            raise GridError("DMI requires A > 0 in every magnetic cell (boundary tilt ~ D/A)")
        self.Kc1 = float(Kc1)
        c1v = np.asarray(c1, dtype=np.float64)
        c1v = c1v / np.linalg.norm(c1v)
        c2v = np.asarray(c2, dtype=np.float64)
        c2v = c2v - np.dot(c2v, c1v) * c1v
        c2v = c2v / np.linalg.norm(c2v)
        self.c1, self.c2 = c1v, c2v
        self.Db = float(Db)
        if self.Db != 0.0 and np.any((self.A <= 0.0) & (self.Ms > 0.0)):
            raise GridError("bulk DMI requires A > 0 in every magnetic cell")
        self._ctx_handle = None
        self._keep = []
        self._n_magnetic = None

    @property
    def mask(self) -> np.ndarray:
        return self.Ms > 0.0

    @property
    def n_magnetic(self) -> int:
        # cached: the material is fixed once built (the device context holds a
        # copy), and at 512^3 the count is 90 ms of host work per run_until
        if self._n_magnetic is None:
            self._n_magnetic = int(np.count_nonzero(self.mask))
        return self._n_magnetic

    def gamma_L(self) -> np.ndarray:
        return self.gamma / (1.0 + self.alpha ** 2)

    def masked(self, per_cell: np.ndarray) -> np.ndarray:
        return np.where(self.mask, per_cell, 0.0)

    # ---- device context -------------------------------------------------
    def _ctx(self):
        """The device context of this material (created on first use)."""
        if self._ctx_handle is not None:
            return self._ctx_handle
        lib = L.load()
        m = L.Material()
        keep = []

        def put(uniform, arr, name):
            if uniform is not None:
                setattr(m, name, uniform)
                return None
            a = np.ascontiguousarray(arr, dtype=np.float64)
            keep.append(a)
            return L.dptr(a)

        m.Ms_cell = put(self._Ms_u, self.Ms, "Ms")
        m.A_cell = put(self._A_u, self.A, "A")
        m.Ku_cell = put(self._Ku_u, self.Ku, "Ku")
        m.D_cell = put(self._D_u, self.D, "D")
        m.alpha_cell = put(self._alpha_u, self.alpha, "alpha")
        m.gamma = self.gamma
        if self._eK_u is not None:
            m.eK = (C.c_double * 3)(*self._eK_u)
            m.eK_cell = None
        else:
            a = np.ascontiguousarray(self.eK)
            keep.append(a)
            m.eK_cell = L.dptr(a)
        m.Kc1 = self.Kc1
        m.c1 = (C.c_double * 3)(*self.c1)
        m.c2 = (C.c_double * 3)(*self.c2)
        m.Db = self.Db
        h = C.c_void_p()
        L.check(lib.mxb_ctx_create(C.byref(self.grid._c()), C.byref(m), L.device(), C.byref(h)),
                "mxb_ctx_create")
        self._ctx_handle = _Ctx(h)
        return self._ctx_handle


class _Ctx:
    """Owner of an mxb_ctx handle."""

    def __init__(self, h):
        self.h = h

    def __del__(self):
        try:
            if self.h:
                L.load().mxb_ctx_destroy(self.h)
        except Exception:
            pass

    def call(self, name, *args):
        lib = L.load()
        lib.mxb_ctx_set_exact(self.h, 1 if L.exact() else 0)
        return getattr(lib, name)(self.h, *args)


def _raise_dead(grid: GridSpec, flat: int):
    i = flat % grid.nx
    j = (flat // grid.nx) % grid.ny
    k = flat // (grid.nx * grid.ny)
    raise RenormalizeError(f"cell (i={i}, j={j}, k={k}) [flat {flat}] has Ms > 0 but |M| = 0")


def renormalize(m: VectorField3, mat: MaterialMap) -> None:
    """Rescale M in place to |M| = Ms, zero vacuum, on the GPU (grid.py:178-200)."""
    ctx = mat._ctx()
    data = m.data
    if not data.flags["C_CONTIGUOUS"]:
        data = np.ascontiguousarray(data)
    dead = C.c_int64(-1)
    rc = ctx.call("mxb_renormalize", L.dptr(data), C.byref(dead))
    if rc == L.EDEAD:
        _raise_dead(m.grid, int(dead.value))
    L.check(rc, "renormalize")
    if data is not m.data:
        m.data[...] = data


def mean_normalized(m: VectorField3, mat: MaterialMap) -> np.ndarray:
    """<M/Ms> over magnetic cells, reduced on the GPU (grid.py:203-214)."""
    if mat.n_magnetic == 0:
        raise GridError("mean_normalized: no magnetic cells (all Ms == 0)")
    out = np.zeros(3)
    L.check(mat._ctx().call("mxb_mean_normalized", L.dptr(np.ascontiguousarray(m.data)),
                            L.dptr(out)), "mean_normalized")
    return out


def ghost_fill(m: VectorField3, mat: MaterialMap, mode: str = "neumann") -> np.ndarray:
    """Ghost-padded copy (grid.py:238-298).  A host utility for analysis and
    tests; the stencil kernels apply the boundary rules in-register instead."""
    if mode not in ("neumann", "dmi", "periodic"):
        raise GridError(f"unknown ghost mode {mode!r}")
    g = m.grid
    out = np.zeros((3, g.nz + 2, g.ny + 2, g.nx + 2))
    out[:, 1:-1, 1:-1, 1:-1] = m.data
    d = (g.dx, g.dy, g.dz)
    for k in range(3):
        ax = 3 - k
        inner = [slice(None), slice(1, -1), slice(1, -1), slice(1, -1)]

        def sl(pos):
            s = list(inner)
            s[ax] = pos
            return tuple(s)

        lo_i, hi_i, lo_g, hi_g = sl(slice(1, 2)), sl(slice(-2, -1)), sl(slice(0, 1)), sl(slice(-1, None))
        if mode == "periodic":
            out[lo_g], out[hi_g] = out[hi_i], out[lo_i]
            continue
        lo, hi = out[lo_i].copy(), out[hi_i].copy()
        if mode == "neumann" or k == 2:
            out[lo_g], out[hi_g] = lo, hi
            continue
        cax = ax - 1
        cs_lo = [slice(None)] * 3
        cs_hi = [slice(None)] * 3
        cs_lo[cax], cs_hi[cax] = slice(0, 1), slice(-1, None)
        for bnd, cs, sign, dst in ((lo, cs_lo, -1.0, lo_g), (hi, cs_hi, 1.0, hi_g)):
            Dv, Av = mat.D[tuple(cs)], mat.A[tuple(cs)]
            with np.errstate(invalid="ignore", divide="ignore"):
                p = np.where(Av > 0.0, -Dv / (2.0 * Av), 0.0)
            slope = np.zeros_like(bnd)
            if k == 0:
                slope[0], slope[2] = p * bnd[2], -p * bnd[0]
            else:
                slope[1], slope[2] = p * bnd[2], -p * bnd[1]
            out[dst] = bnd + sign * d[k] * slope
    return out
