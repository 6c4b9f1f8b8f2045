"""Local effective-field terms and energies (reference: fields.py).

Each operator keeps the reference constructor/call signature
(``op = ExchangeOperator(mat, ghost_mode, plan); h = op(mdata)``) and runs the
fused stencil kernel (csrc/stencil.cu) restricted to its own term.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .grid import MU0, GridSpec, MaterialMap, VectorField3  # noqa: F401

GHOST_MODES = ("neumann", "dmi", "periodic")


class _StencilPlan:
    """Boundary-mode holder (fields.py:49-92).  The validity masks and face
    coefficients are recomputed in-register by the kernel from Ms and A."""

    def __init__(self, mat: MaterialMap, ghost_mode: str):
        if ghost_mode not in GHOST_MODES:
            raise ValueError(f"unknown ghost mode {ghost_mode!r}")
        self.mat = mat
        self.mode = ghost_mode


def _term(mat: MaterialMap, term: int, mode: str, mdata: np.ndarray) -> np.ndarray:
    m = np.ascontiguousarray(mdata, dtype=np.float64)
    if m.shape != (3,) + mat.grid.shape:
        raise ValueError(f"field shape {m.shape} does not match grid {(3,) + mat.grid.shape}")
    h = np.empty_like(m)
    L.check(mat._ctx().call("mxb_term_field", term, L.GHOST[mode], L.dptr(m), L.dptr(h)), "term")
    return h


class ExchangeOperator:
    """H_exch = (2/(mu0 Ms^2)) div(A grad M), flux form (fields.py:102-127)."""

    def __init__(self, mat: MaterialMap, ghost_mode: str = "neumann",
                 plan: _StencilPlan | None = None):
        self.mat = mat
        self.plan = plan or _StencilPlan(mat, ghost_mode)

    def __call__(self, mdata: np.ndarray) -> np.ndarray:
        return _term(self.mat, L.TERM_EXCHANGE, self.plan.mode, mdata)


class DmiOperator:
    """Interfacial DMI field (fields.py:130-151)."""

    def __init__(self, mat: MaterialMap, ghost_mode: str = "dmi",
                 plan: _StencilPlan | None = None):
        self.mat = mat
        self.plan = plan or _StencilPlan(mat, ghost_mode)

    def __call__(self, mdata: np.ndarray) -> np.ndarray:
        return _term(self.mat, L.TERM_DMI, self.plan.mode, mdata)


class AnisotropyOperator:
    """Uniaxial anisotropy H = (2Ku/(mu0 Ms^2))(M.eK)eK (fields.py:154-163)."""

    def __init__(self, mat: MaterialMap):
        self.mat = mat

    def __call__(self, mdata: np.ndarray) -> np.ndarray:
        return _term(self.mat, L.TERM_ANISOTROPY, "neumann", mdata)


class CubicAnisotropyOperator:
    """Cubic anisotropy (extension; parity unpinned):
    E = Kc1 (a1^2 a2^2 + a2^2 a3^2 + a3^2 a1^2), a_i = m.c_i."""

    def __init__(self, mat: MaterialMap):
        self.mat = mat

    def __call__(self, mdata: np.ndarray) -> np.ndarray:
        return _term(self.mat, L.TERM_CUBIC, "neumann", mdata)


class BulkDmiOperator:
    """Bulk DMI (extension; parity unpinned):
    E = Db m.(curl m), H = -(2 Db/(mu0 Ms^2)) curl M."""

    def __init__(self, mat: MaterialMap):
        self.mat = mat

    def __call__(self, mdata: np.ndarray) -> np.ndarray:
        return _term(self.mat, L.TERM_BULK_DMI, "neumann", mdata)


def exchange_field(m: VectorField3, mat: MaterialMap, ghost_mode: str = "neumann") -> np.ndarray:
    return ExchangeOperator(mat, ghost_mode)(m.data)


def dmi_field(m: VectorField3, mat: MaterialMap, ghost_mode: str = "dmi") -> np.ndarray:
    return DmiOperator(mat, ghost_mode)(m.data)


def anisotropy_field(m: VectorField3, mat: MaterialMap) -> np.ndarray:
    return AnisotropyOperator(mat)(m.data)


def cubic_anisotropy_field(m: VectorField3, mat: MaterialMap) -> np.ndarray:
    return CubicAnisotropyOperator(mat)(m.data)


def bulk_dmi_field(m: VectorField3, mat: MaterialMap) -> np.ndarray:
    return BulkDmiOperator(mat)(m.data)


def uniform_bias(vec) -> np.ndarray:
    return np.asarray(vec, dtype=np.float64)


@dataclass
class EnergyBreakdown:
    """Energy densities in J/m^3 averaged over magnetic cells (fields.py:180-191)."""

    e_demag: float
    e_exch: float
    e_anis: float
    e_zeeman: float

    @property
    def e_total(self) -> float:
        return self.e_demag + self.e_exch + self.e_anis + self.e_zeeman


def energy_breakdown(m: VectorField3, mat: MaterialMap, h_demag: np.ndarray | None = None,
                     h_bias: np.ndarray | None = None, ghost_mode: str = "neumann",
                     plan: _StencilPlan | None = None) -> EnergyBreakdown:
    """Energy densities of the state, reduced on the GPU (fields.py:200-242)."""
    if not np.any(mat.mask):
        raise ValueError("energy_breakdown: no magnetic cells")
    mode = plan.mode if plan is not None else ghost_mode
    mask = 0
    b = L.Bias()
    keep = []
    if h_demag is not None:
        hd = np.ascontiguousarray(h_demag, dtype=np.float64)
        keep.append(hd)
        b.demag_field = L.dptr(hd)
        mask |= L.TERM_DEMAG
    if h_bias is not None:
        hb = np.asarray(h_bias, dtype=np.float64)
        mask |= L.TERM_BIAS
        if hb.shape == (3,):
            b.vec = (C.c_double * 3)(*hb)
        else:
            hb = np.ascontiguousarray(np.broadcast_to(hb, (3,) + mat.grid.shape))
            keep.append(hb)
            b.field = L.dptr(hb)
    t = L.Terms(mask, L.GHOST[mode], 1, 1)
    out = np.zeros(4)
    md = np.ascontiguousarray(m.data)
    L.check(mat._ctx().call("mxb_energies", None, C.byref(t), C.byref(b), L.dptr(md),
                            L.dptr(out)), "energies")
    return EnergyBreakdown(float(out[0]), float(out[1]), float(out[2]), float(out[3]))
