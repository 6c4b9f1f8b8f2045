"""CPU oracle for the MagneX H_eff + LLG hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package ``magnex`` 0.1.0
(`/root/reference/pkg/src/magnex`), kept bit-for-bit faithful in operation
order so that it reproduces the reference's float64 results exactly on the
same inputs.  It is imported only by ``tests/``, ``__graft_entry__.smoke()``
and the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py``, and
there only as the checker or the timed CPU baseline -- never by the product
package ``paper_2602_12242_b200``.

Parity pinning: ``tests/test_oracle_golden.py`` checks every function here
against golden vectors produced by running the reference itself
(``tests/golden/make_golden.py``, numpy 2.3.5 / scipy 1.18.1).  The FFT is the
third-party boundary: scipy.fft (pocketfft C++, scipy 1.18.1 wheel), called
exactly as the reference calls it (``demag.py:191,209,215``).

Cubic anisotropy and bulk DMI (``cubic_anisotropy_field``/``bulk_dmi_field``)
have no reference implementation: they are *parity unpinned*
restatements of the standard continuum formulas and are checked by analytic
properties only.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field as dc_field

import numpy as np
import scipy.fft as sfft

MU0 = 4.0e-7 * math.pi          # grid.py:17
GAMMA = -1.759e11               # grid.py:18
BLOWUP_DRIFT = 0.10             # llg.py:51
DIPOLE_SWITCH_DIAGONALS = 60.0  # demag.py:29
MIX = ((0, 1, 2), (1, 3, 4), (2, 4, 5))  # demag.py:33-34 (XX,XY,XZ,YY,YZ,ZZ)


class OracleRenormalizeError(ValueError):
    pass


class OracleBlowup(RuntimeError):
    def __init__(self, step, t, drift):
        super().__init__(f"blow-up at step {step}")
        self.step, self.t, self.drift = step, t, drift


# ----------------------------------------------------------------------------
# material (grid.py:110-175)
# ----------------------------------------------------------------------------

def _cellwise(v, shape):
    a = np.asarray(v, dtype=np.float64)
    if a.ndim == 0:
        return np.full(shape, float(a))
    assert a.shape == shape
    return np.ascontiguousarray(a)


@dataclass
class Mat:
    """Per-cell material in the reference layout (grid.py:119-158)."""
    dims: tuple          # (nx, ny, nz)
    cell: tuple          # (dx, dy, dz)
    Ms: np.ndarray
    A: np.ndarray
    Ku: np.ndarray
    D: np.ndarray
    alpha: np.ndarray
    eK: np.ndarray
    gamma: float = GAMMA
    Kc1: np.ndarray | None = None     # cubic K1 (unpinned extension)
    c1: np.ndarray | None = None      # cubic axis 1 (3,)
    c2: np.ndarray | None = None      # cubic axis 2 (3,)
    Db: np.ndarray | None = None      # bulk DMI constant (unpinned extension)

    @property
    def shape(self):
        nx, ny, nz = self.dims
        return (nz, ny, nx)

    @property
    def mask(self):
        return self.Ms > 0.0


def make_mat(dims, cell, Ms, A=0.0, Ku=0.0, eK=(0.0, 0.0, 1.0), D=0.0, alpha=0.0,
             gamma=GAMMA, Kc1=0.0, c1=(1.0, 0.0, 0.0), c2=(0.0, 1.0, 0.0), Db=0.0):
    nx, ny, nz = dims
    shape = (nz, ny, nx)
    e = np.asarray(eK, dtype=np.float64)
    if e.shape == (3,):
        ek = np.empty((3,) + shape)
        for c in range(3):
            ek[c] = e[c]
    else:
        ek = np.ascontiguousarray(e)
    n = np.sqrt(np.einsum("cijk,cijk->ijk", ek, ek))          # grid.py:147
    with np.errstate(invalid="ignore", divide="ignore"):
        ek = np.where(n > 0.0, ek / n, 0.0)                      # grid.py:152
    c1v = np.asarray(c1, dtype=np.float64)
    c1v = c1v / np.linalg.norm(c1v)
    c2v = np.asarray(c2, dtype=np.float64)
    c2v = c2v - np.dot(c2v, c1v) * c1v
    c2v = c2v / np.linalg.norm(c2v)
    return Mat(tuple(dims), tuple(cell), _cellwise(Ms, shape), _cellwise(A, shape),
               _cellwise(Ku, shape), _cellwise(D, shape), _cellwise(alpha, shape), ek,
               float(gamma), _cellwise(Kc1, shape), c1v, c2v, _cellwise(Db, shape))


# ----------------------------------------------------------------------------
# per-cell primitives (grid.py:178-235)
# ----------------------------------------------------------------------------

def renormalize(m: np.ndarray, mat: Mat) -> np.ndarray:
    """Return M rescaled to |M| = Ms (grid.py:178-200); raises on dead cells."""
    n2 = np.einsum("cijk,cijk->ijk", m, m)
    mask = mat.mask
    dead = mask & (n2 == 0.0)
    if dead.any():
        k, j, i = (int(v[0]) for v in np.nonzero(dead))
        nx, ny, _ = mat.dims
        raise OracleRenormalizeError(f"cell (i={i}, j={j}, k={k}) [flat {i + nx * (j + ny * k)}]")
    ms2 = mat.Ms * mat.Ms
    stale = mask & (np.abs(n2 - ms2) > 1e-15 * ms2)              # grid.py:196
    with np.errstate(invalid="ignore", divide="ignore"):
        s = np.where(stale, mat.Ms / np.sqrt(np.where(stale, n2, 1.0)), 1.0)
        s = np.where(mask, s, 0.0)
    return m * s


def mean_normalized(m: np.ndarray, mat: Mat) -> np.ndarray:
    """<M/Ms> over magnetic cells (grid.py:203-214)."""
    mask = mat.mask
    cnt = int(np.count_nonzero(mask))
    if cnt == 0:
        raise ValueError("no magnetic cells")
    with np.errstate(invalid="ignore", divide="ignore"):
        q = m / np.where(mask, mat.Ms, 1.0)
    return np.array([q[c][mask].sum() / cnt for c in range(3)])


def boundary_slope(m: np.ndarray, mat: Mat, k: int) -> np.ndarray:
    """Interfacial-DMI natural-boundary slope dM/dx_k (grid.py:217-235)."""
    s = np.zeros_like(m)
    if k == 2:
        return s
    with np.errstate(invalid="ignore", divide="ignore"):
        p = np.where(mat.A > 0.0, -mat.D / (2.0 * mat.A), 0.0)
    if k == 0:
        s[0] = p * m[2]
        s[2] = -p * m[0]
    else:
        s[1] = p * m[2]
        s[2] = -p * m[1]
    return s


# ----------------------------------------------------------------------------
# stencil plan (fields.py:23-92)
# ----------------------------------------------------------------------------

def _neighbour(a: np.ndarray, k: int, step: int, periodic: bool) -> np.ndarray:
    """Value of the step-neighbour along cartesian axis k; domain faces repeat
    the face value (fields.py:23-46)."""
    ax = a.ndim - 1 - k
    if periodic:
        return np.roll(a, -step, axis=ax)
    n = a.shape[ax]
    idx = np.clip(np.arange(n) + step, 0, n - 1)
    return np.take(a, idx, axis=ax)


class Plan:
    """Neighbour validity and harmonic face coefficients (fields.py:49-92)."""

    def __init__(self, mat: Mat, mode: str):
        assert mode in ("neumann", "dmi", "periodic")
        self.mat, self.mode = mat, mode
        per = mode == "periodic"
        mask = mat.mask
        self.valid, self.face = {}, {}
        for k in range(3):
            ax = 2 - k
            n = mask.shape[ax]
            for step in (1, -1):
                v = _neighbour(mask, k, step, per)
                if not per:
                    v = v.copy()
                    sl = [slice(None)] * 3
                    sl[ax] = slice(n - 1, n) if step > 0 else slice(0, 1)
                    v[tuple(sl)] = False
                self.valid[(k, step)] = v
                An = _neighbour(mat.A, k, step, per)
                tot = mat.A + An
                with np.errstate(invalid="ignore", divide="ignore"):
                    harm = np.where(tot > 0.0, 2.0 * mat.A * An / np.where(tot > 0.0, tot, 1.0), 0.0)
                self.face[(k, step)] = np.where(v, harm, mat.A)

    def nb(self, m: np.ndarray, k: int, step: int) -> np.ndarray:
        per = self.mode == "periodic"
        raw = _neighbour(m, k, step, per)
        if per:
            return raw
        if self.mode == "neumann":
            ghost = m
        else:
            d = self.mat.cell[k]
            ghost = m + step * d * boundary_slope(m, self.mat, k)
        return np.where(self.valid[(k, step)], raw, ghost)


def field_prefactor(mat: Mat) -> np.ndarray:
    """2/(mu0 Ms^2) on magnetic cells (fields.py:95-99)."""
    mask = mat.mask
    with np.errstate(invalid="ignore", divide="ignore"):
        return np.where(mask, 2.0 / (MU0 * np.where(mask, mat.Ms, 1.0) ** 2), 0.0)


# ----------------------------------------------------------------------------
# local field terms (fields.py:102-163)
# ----------------------------------------------------------------------------

def exchange_field(m, mat: Mat, plan: Plan) -> np.ndarray:
    """Flux-form exchange (fields.py:112-127)."""
    acc = np.zeros_like(m)
    for k in range(3):
        if mat.dims[k] <= 1:
            continue
        d = mat.cell[k]
        up, dn = plan.nb(m, k, 1), plan.nb(m, k, -1)
        acc += (plan.face[(k, 1)] * (up - m) - plan.face[(k, -1)] * (m - dn)) / (d * d)
    h = field_prefactor(mat) * acc
    h[:, ~mat.mask] = 0.0
    return h


def dmi_field(m, mat: Mat, plan: Plan) -> np.ndarray:
    """Interfacial DMI (fields.py:142-151)."""
    dx, dy, _ = mat.cell
    gx = (plan.nb(m, 0, 1) - plan.nb(m, 0, -1)) / (2 * dx)
    gy = (plan.nb(m, 1, 1) - plan.nb(m, 1, -1)) / (2 * dy)
    p = field_prefactor(mat) * mat.D
    h = np.empty_like(m)
    h[0] = p * gx[2]
    h[1] = p * gy[2]
    h[2] = -p * (gx[0] + gy[1])
    h[:, ~mat.mask] = 0.0
    return h


def anisotropy_field(m, mat: Mat) -> np.ndarray:
    """Uniaxial anisotropy (fields.py:161-163)."""
    p = field_prefactor(mat) * mat.Ku
    return (p * np.einsum("cijk,cijk->ijk", m, mat.eK)) * mat.eK


def cubic_anisotropy_field(m, mat: Mat) -> np.ndarray:
    """Cubic anisotropy, E = K1 (a1^2 a2^2 + a2^2 a3^2 + a3^2 a1^2), a_i = m.c_i.

    PARITY UNPINNED (no reference implementation).
    H = -(2 K1/(mu0 Ms)) sum_i a_i (a_j^2 + a_k^2) c_i, with m = M/Ms.
    """
    c1, c2 = mat.c1, mat.c2
    c3 = np.cross(c1, c2)
    mask = mat.mask
    with np.errstate(invalid="ignore", divide="ignore"):
        inv = np.where(mask, 1.0 / np.where(mask, mat.Ms, 1.0), 0.0)
    mn = m * inv
    a = [np.einsum("c,cijk->ijk", c, mn) for c in (c1, c2, c3)]
    with np.errstate(invalid="ignore", divide="ignore"):
        p = np.where(mask, -2.0 * mat.Kc1 / (MU0 * np.where(mask, mat.Ms, 1.0)), 0.0)
    h = np.zeros_like(m)
    for i, ci in enumerate((c1, c2, c3)):
        j, k = (i + 1) % 3, (i + 2) % 3
        w = p * a[i] * (a[j] ** 2 + a[k] ** 2)
        for c in range(3):
            h[c] += w * ci[c]
    return h


def bulk_dmi_field(m, mat: Mat) -> np.ndarray:
    """Bulk DMI, E = Db m.(curl m); H = -(2 Db/(mu0 Ms^2)) curl M.

    PARITY UNPINNED (no reference implementation).
    Central differences; a missing neighbour (domain face or vacuum) takes the
    bulk-DMI natural-boundary ghost M + step*d*(Db/2A)(e_k x M); singleton axes
    therefore contribute the exact boundary slope.
    """
    mask = mat.mask
    nx, ny, nz = mat.dims
    curl_parts = []
    grads = []
    for k in range(3):
        d = mat.cell[k]
        ek = np.zeros(3)
        ek[k] = 1.0
        with np.errstate(invalid="ignore", divide="ignore"):
            pr = np.where(mat.A > 0.0, mat.Db / (2.0 * mat.A), 0.0)
        cr = np.empty_like(m)                   # e_k x M
        cr[0] = ek[1] * m[2] - ek[2] * m[1]
        cr[1] = ek[2] * m[0] - ek[0] * m[2]
        cr[2] = ek[0] * m[1] - ek[1] * m[0]
        slope = pr * cr
        vals = []
        for step in (1, -1):
            raw = _neighbour(m, k, step, False)
            v = _neighbour(mask, k, step, False).copy()
            ax = 2 - k
            n = mask.shape[ax]
            sl = [slice(None)] * 3
            sl[ax] = slice(n - 1, n) if step > 0 else slice(0, 1)
            v[tuple(sl)] = False
            vals.append(np.where(v, raw, m + step * d * slope))
        grads.append((vals[0] - vals[1]) / (2 * d))
    gx, gy, gz = grads
    curl = np.empty_like(m)
    curl[0] = gy[2] - gz[1]
    curl[1] = gz[0] - gx[2]
    curl[2] = gx[1] - gy[0]
    p = -field_prefactor(mat) * mat.Db
    h = p * curl
    h[:, ~mask] = 0.0
    return h


# ----------------------------------------------------------------------------
# demagnetisation (demag.py:37-216)
# ----------------------------------------------------------------------------

def _guarded(num, den):
    ok = den != 0
    return np.where(ok, num / np.where(ok, den, 1), 0.0)


def newell_f(x, y, z):
    """Diagonal-element antiderivative (demag.py:37-50)."""
    x, y, z = np.abs(x), np.abs(y), np.abs(z)
    xx, yy, zz = x * x, y * y, z * z
    r = np.sqrt(xx + yy + zz)
    rxz = np.sqrt(xx + zz)
    rxy = np.sqrt(xx + yy)
    with np.errstate(invalid="ignore", divide="ignore"):
        a = 0.5 * y * (zz - xx) * np.arcsinh(np.where(rxz > 0, y / np.where(rxz > 0, rxz, 1), 0))
        b = 0.5 * z * (yy - xx) * np.arcsinh(np.where(rxy > 0, z / np.where(rxy > 0, rxy, 1), 0))
        xr = x * r
        c = -x * y * z * np.arctan(np.where(xr > 0, y * z / np.where(xr > 0, xr, 1), 0))
    d = (2 * xx - yy - zz) * r / 6.0
    return a + b + c + d


def newell_g(x, y, z):
    """Off-diagonal antiderivative (demag.py:53-77)."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    z = np.abs(z)
    xx, yy, zz = x * x, y * y, z * z
    r = np.sqrt(xx + yy + zz)
    rxy, ryz, rxz = np.sqrt(xx + yy), np.sqrt(yy + zz), np.sqrt(xx + zz)
    with np.errstate(invalid="ignore", divide="ignore"):
        t1 = x * y * z * np.arcsinh(_guarded(z, rxy))
        t2 = (y / 6.0) * (3 * zz - yy) * np.arcsinh(_guarded(x, ryz))
        t3 = (x / 6.0) * (3 * zz - xx) * np.arcsinh(_guarded(y, rxz))
        t4 = -(zz * z / 6.0) * np.arctan(_guarded(x * y, z * r))
        t5 = -(z * yy / 2.0) * np.arctan(_guarded(x * z, y * r))
        t6 = -(z * xx / 2.0) * np.arctan(_guarded(y * z, x * r))
    t7 = -x * y * r / 3.0
    return t1 + t2 + t3 + t4 + t5 + t6 + t7


def _d2(a, ax):
    n = a.shape[ax]
    lo = np.take(a, range(0, n - 2), axis=ax)
    mid = np.take(a, range(1, n - 1), axis=ax)
    hi = np.take(a, range(2, n), axis=ax)
    return hi - 2.0 * mid + lo                    # demag.py:80-87


def tensor_elements(nx, ny, nz, dx, dy, dz) -> np.ndarray:
    """(6, 2nz-1, 2ny-1, 2nx-1) cell-pair tensor (demag.py:90-120)."""
    s = (dx * dy * dz) ** (1.0 / 3.0)
    ux, uy, uz = dx / s, dy / s, dz / s
    Zg, Yg, Xg = np.meshgrid(np.arange(-nz, nz + 1) * uz, np.arange(-ny, ny + 1) * uy,
                             np.arange(-nx, nx + 1) * ux, indexing="ij")
    jobs = ((newell_f, (Xg, Yg, Zg)), (newell_g, (Xg, Yg, Zg)), (newell_g, (Xg, Zg, Yg)),
            (newell_f, (Yg, Zg, Xg)), (newell_g, (Yg, Zg, Xg)), (newell_f, (Zg, Xg, Yg)))
    out = np.empty((6, 2 * nz - 1, 2 * ny - 1, 2 * nx - 1))
    for c, (fn, args) in enumerate(jobs):
        F = fn(*args)
        for ax in (0, 1, 2):
            F = _d2(F, ax)
        out[c] = F / (4.0 * np.pi)
    _dipole_far(out, nx, ny, nz, ux, uy, uz)
    return out


def _dipole_far(n6, nx, ny, nz, ux, uy, uz):
    """Point-dipole elements beyond 60 cell diagonals (demag.py:123-141)."""
    diag = np.sqrt(ux * ux + uy * uy + uz * uz)
    Zg, Yg, Xg = np.meshgrid(np.arange(-(nz - 1), nz) * uz, np.arange(-(ny - 1), ny) * uy,
                             np.arange(-(nx - 1), nx) * ux, indexing="ij")
    r2 = Xg * Xg + Yg * Yg + Zg * Zg
    far = r2 > (DIPOLE_SWITCH_DIAGONALS * diag) ** 2
    if not far.any():
        return
    x, y, z, q = Xg[far], Yg[far], Zg[far], r2[far]
    r5 = q ** 2.5
    c = 1.0 / (4.0 * np.pi)
    n6[0][far] = c * (3 * x * x - q) / r5
    n6[3][far] = c * (3 * y * y - q) / r5
    n6[5][far] = c * (3 * z * z - q) / r5
    n6[1][far] = c * 3 * x * y / r5
    n6[2][far] = c * 3 * x * z / r5
    n6[4][far] = c * 3 * y * z / r5


def padded_dims(nx, ny, nz):
    """(pz, py, px), 2n or 1 (demag.py:152-155)."""
    return (2 * nz if nz > 1 else 1, 2 * ny if ny > 1 else 1, 2 * nx if nx > 1 else 1)


def pack_wraparound(n6, nx, ny, nz) -> np.ndarray:
    """Displacement d -> index d mod p (demag.py:158-166)."""
    pz, py, px = padded_dims(nx, ny, nz)
    out = np.zeros((6, pz, py, px))
    iz = np.arange(-(nz - 1), nz) % pz
    iy = np.arange(-(ny - 1), ny) % py
    ix = np.arange(-(nx - 1), nx) % px
    out[np.ix_(range(6), iz, iy, ix)] = n6
    return out


def packed_tensor(nx, ny, nz, dx, dy, dz) -> np.ndarray:
    return pack_wraparound(tensor_elements(nx, ny, nz, dx, dy, dz), nx, ny, nz)


def kernel_spectra(packed: np.ndarray, workers: int = 1) -> np.ndarray:
    """6 r2c spectra of the packed tensor (demag.py:190-195)."""
    return np.stack([sfft.rfftn(packed[c], s=packed.shape[1:], workers=workers)
                     for c in range(6)])


def demag_field(spectra: np.ndarray, m: np.ndarray, workers: int | None = None) -> np.ndarray:
    """Zero-padded FFT convolution H = N * M (demag.py:203-216)."""
    _, nz, ny, nx = m.shape
    pad = padded_dims(nx, ny, nz)
    buf = np.zeros((3,) + pad)
    buf[:, :nz, :ny, :nx] = m
    mh = [sfft.rfftn(buf[c], s=pad, workers=workers) for c in range(3)]
    h = np.empty_like(m)
    for a in range(3):
        acc = spectra[MIX[a][0]] * mh[0]
        acc += spectra[MIX[a][1]] * mh[1]
        acc += spectra[MIX[a][2]] * mh[2]
        h[a] = sfft.irfftn(acc, s=pad, workers=workers)[:nz, :ny, :nx]
    return h


def demag_direct(m: np.ndarray, n6: np.ndarray) -> np.ndarray:
    """O(N^2) direct sum over source cells (demag.py:225-248)."""
    _, nz, ny, nx = m.shape
    h = np.zeros_like(m)
    for qz in range(nz):
        for qy in range(ny):
            for qx in range(nx):
                src = m[:, qz, qy, qx]
                if not src.any():
                    continue
                blk = n6[:, nz - 1 - qz:2 * nz - 1 - qz, ny - 1 - qy:2 * ny - 1 - qy,
                         nx - 1 - qx:2 * nx - 1 - qx]
                for a in range(3):
                    h[a] += (blk[MIX[a][0]] * src[0] + blk[MIX[a][1]] * src[1]
                             + blk[MIX[a][2]] * src[2])
    return h


# ----------------------------------------------------------------------------
# torque, RHS assembly, steppers (llg.py:64-203, integrators.py:43-64)
# ----------------------------------------------------------------------------

def llg_rhs(m, h, mat: Mat, precession=True, damping=True) -> np.ndarray:
    """mu0 gL M x H + (alpha mu0 gL / Ms) M x (M x H), masked damping (llg.py:64-74)."""
    gl = MU0 * (mat.gamma / (1.0 + mat.alpha ** 2))
    mxh = np.cross(m, h, axisa=0, axisb=0, axisc=0)
    out = np.zeros_like(m)
    if precession:
        out += gl * mxh
    if damping:
        mask = mat.mask
        coef = np.where(mask, gl * mat.alpha / np.where(mask, mat.Ms, 1.0), 0.0)
        out += coef * np.cross(m, mxh, axisa=0, axisb=0, axisc=0)
    return out


@dataclass
class Terms:
    """Which H_eff terms are on, in the reference's accumulation order
    exchange, anisotropy, dmi, demag, bias (llg.py:112-125,145-149)."""
    exchange: bool = True
    anisotropy: bool = False
    dmi: bool = False
    spectra: np.ndarray | None = None     # demag kernel spectra or None
    bias: object = None                   # None, 3-vector, field, or callable(t)
    precession: bool = True
    damping: bool = True
    ghost_mode: str | None = None
    cubic: bool = False                   # unpinned extension (after anisotropy)
    bulk_dmi: bool = False                # unpinned extension (after dmi)

    def mode(self):
        return self.ghost_mode or ("dmi" if self.dmi else "neumann")


def bias_at(terms: Terms, t: float):
    if terms.bias is None:
        return None
    b = terms.bias(t) if callable(terms.bias) else terms.bias
    return np.asarray(b, dtype=np.float64)


def h_eff(t, m, mat: Mat, terms: Terms, plan: Plan | None = None) -> np.ndarray:
    plan = plan or Plan(mat, terms.mode())
    h = np.zeros_like(m)
    if terms.exchange:
        h += exchange_field(m, mat, plan)
    if terms.anisotropy:
        h += anisotropy_field(m, mat)
    if terms.cubic:
        h += cubic_anisotropy_field(m, mat)
    if terms.dmi:
        h += dmi_field(m, mat, plan)
    if terms.bulk_dmi:
        h += bulk_dmi_field(m, mat)
    if terms.spectra is not None:
        h += demag_field(terms.spectra, m)
    b = bias_at(terms, t)
    if b is not None:
        h += b.reshape(3, 1, 1, 1) if b.shape == (3,) else b
    return h


def rhs_total(t, m, mat: Mat, terms: Terms, plan: Plan | None = None) -> np.ndarray:
    return llg_rhs(m, h_eff(t, m, mat, terms, plan), mat, terms.precession, terms.damping)


def euler_step(y, t, dt, f):
    return y + dt * f(t, y)                        # integrators.py:43-45


def rk4_step(y, t, dt, f, post=None):
    """Classical RK4 with post-stage hook on y2..y4 (integrators.py:48-64)."""
    h2 = 0.5 * dt
    k1 = f(t, y)
    y2 = y + h2 * k1
    y2 = post(y2) if post else y2
    k2 = f(t + h2, y2)
    y3 = y + h2 * k2
    y3 = post(y3) if post else y3
    k3 = f(t + h2, y3)
    y4 = y + dt * k3
    y4 = post(y4) if post else y4
    k4 = f(t + dt, y4)
    return y + (dt / 6.0) * (k1 + 2.0 * (k2 + k3) + k4)


# Knoth-Wolke tableau and multirate forcing weights (integrators.py:28-40)
KW3_C = (0.0, 1.0 / 3.0, 3.0 / 4.0)
KW3_A = ((0.0, 0.0, 0.0), (1.0 / 3.0, 0.0, 0.0), (-3.0 / 16.0, 15.0 / 16.0, 0.0))
KW3_B = (1.0 / 6.0, 3.0 / 10.0, 8.0 / 15.0)
MRI_DC = (1.0 / 3.0, 5.0 / 12.0, 1.0 / 4.0)
MRI_W = ((1.0,), (-5.0 / 4.0, 9.0 / 4.0), (17.0 / 12.0, -51.0 / 20.0, 32.0 / 15.0))


def kw3_step(y, t, dt, f, post=None):
    """Three-stage third-order step (integrators.py:67-78)."""
    k1 = f(t, y)
    y2 = y + (dt * KW3_A[1][0]) * k1
    y2 = post(y2) if post else y2
    k2 = f(t + KW3_C[1] * dt, y2)
    y3 = y + dt * (KW3_A[2][0] * k1 + KW3_A[2][1] * k2)
    y3 = post(y3) if post else y3
    k3 = f(t + KW3_C[2] * dt, y3)
    return y + dt * (KW3_B[0] * k1 + KW3_B[1] * k2 + KW3_B[2] * k3)


def substeps(theta):
    """ceil(delta-c / theta) fast substeps per slow phase (integrators.py:81-89)."""
    return tuple(math.ceil(dc / theta - 1e-12) for dc in MRI_DC)


def mri_kw3_step(y, t, dt, f_slow, f_fast, theta=0.1, post=None):
    """Explicit multirate step: 3 slow evaluations, KW3-subcycled fast system
    under piecewise-constant slow forcing (integrators.py:97-128)."""
    n = substeps(theta)
    fs = [f_slow(t, y)]
    v = y
    for ph in range(3):
        w = MRI_W[ph]
        r = w[0] * fs[0]
        for j in range(1, len(w)):
            r = r + w[j] * fs[j]
        h = MRI_DC[ph] * dt / n[ph]
        t0 = t + KW3_C[ph] * dt
        for s in range(n[ph]):
            v = kw3_step(v, t0 + s * h, h, lambda tt, vv, r=r: f_fast(tt, vv) + r, post)
            v = post(v) if post else v
        if ph < 2:
            fs.append(f_slow(t + KW3_C[ph + 1] * dt, v))
    return v


def split_terms(terms: Terms, fast: set):
    """(slow, fast) Terms of a partition (llg.py:127-136,183-189)."""
    import dataclasses
    on = {"exchange": terms.exchange, "anisotropy": terms.anisotropy, "dmi": terms.dmi,
          "demag": terms.spectra is not None, "bias": terms.bias is not None}
    mode = terms.mode()

    def pick(keep):
        return dataclasses.replace(
            terms, exchange=on["exchange"] and "exchange" in keep,
            anisotropy=on["anisotropy"] and "anisotropy" in keep, dmi=on["dmi"] and "dmi" in keep,
            spectra=terms.spectra if "demag" in keep else None,
            bias=terms.bias if "bias" in keep else None, ghost_mode=mode)

    all_terms = set(on)
    return pick(all_terms - fast), pick(fast)


def energies(t, m, mat: Mat, terms: Terms, plan: Plan | None = None):
    """(e_demag, e_exch, e_anis, e_zeeman), means over magnetic cells
    (fields.py:200-242 via llg.py:201-203)."""
    plan = plan or Plan(mat, terms.mode())
    mask = mat.mask
    cnt = np.count_nonzero(mask)

    def mean(x):
        return float(x[mask].sum() / cnt)

    e_dem = 0.0
    if terms.spectra is not None:
        hd = demag_field(terms.spectra, m)
        e_dem = mean(-0.5 * MU0 * np.einsum("cijk,cijk->ijk", m, hd))
    with np.errstate(invalid="ignore", divide="ignore"):
        mn = np.where(mask, m / np.where(mask, mat.Ms, 1.0), 0.0)
    g2 = np.zeros(mat.shape)
    for k in range(3):
        if mat.dims[k] == 1 and plan.mode != "dmi":
            continue
        dk = (plan.nb(mn, k, 1) - plan.nb(mn, k, -1)) / (2 * mat.cell[k])
        g2 += np.einsum("cijk,cijk->ijk", dk, dk)
    e_ex = mean(mat.A * g2)
    pr = np.einsum("cijk,cijk->ijk", mn, mat.eK)
    e_an = mean(mat.Ku * (1.0 - pr ** 2))
    e_ze = 0.0
    b = bias_at(terms, t)
    if b is not None:
        hb = b.reshape(3, 1, 1, 1) if b.shape == (3,) else b
        e_ze = mean(-MU0 * np.einsum("cijk,cijk->ijk", m, np.broadcast_to(hb, m.shape)))
    return e_dem, e_ex, e_an, e_ze


@dataclass
class RunResult:
    m: np.ndarray
    t: float
    step: int
    rows: list = dc_field(default_factory=list)
    stop_reason: str = ""
    final_residual: float = float("nan")
    evals: int = 0


def run(m0, mat: Mat, terms: Terms, method: str, dt: float, *, t0=0.0, step0=0,
        max_time=None, max_steps=None, eq_tol=None, renorm_each_stage=True,
        sample_every=10 ** 9, with_energies=False, theta=0.1, fast=("exchange",)) -> RunResult:
    """Fixed-step driver loop of Simulation.run_until (llg.py:320-379)."""
    plan = Plan(mat, terms.mode())

    def f(t, y):
        return rhs_total(t, y, mat, terms, plan)

    slow_t, fast_t = split_terms(terms, set(fast))

    def f_slow(t, y):
        return rhs_total(t, y, mat, slow_t, plan)

    def f_fast(t, y):
        return rhs_total(t, y, mat, fast_t, plan)

    def post(y):
        return renormalize(y, mat)

    def row(mm, t):
        mb = mean_normalized(mm, mat)
        r = {"t": t, "mx": mb[0], "my": mb[1], "mz": mb[2]}
        if with_energies:
            e = energies(t, mm, mat, terms, plan)
            r.update(e_demag=e[0], e_exch=e[1], e_anis=e[2], e_total=e[0] + e[1] + e[2] + e[3])
        return r

    n_total = None
    if max_time is not None:
        n_total = max(int(round((max_time - t0) / dt)), 0)
    if max_steps is not None:
        n_total = max_steps if n_total is None else min(n_total, max_steps)
    res = RunResult(m=m0.copy(), t=t0, step=step0)
    res.rows.append(row(res.m, res.t))
    prev = mean_normalized(res.m, mat)
    reason = "max_time" if max_time is not None else "max_steps"
    if n_total is not None and max_steps is not None and n_total == max_steps:
        reason = "max_steps"
    mask = mat.mask
    k = 0
    hit_eq = False
    while k < n_total:
        if method == "euler":
            y = euler_step(res.m, res.t, dt, f)
            res.evals += 1
        elif method == "rk4":
            y = rk4_step(res.m, res.t, dt, f, post if renorm_each_stage else None)
            res.evals += 4
        elif method == "mri-kw3":
            y = mri_kw3_step(res.m, res.t, dt, f_slow, f_fast, theta,
                             post if renorm_each_stage else None)
            res.evals += 3
        else:
            raise ValueError(method)
        nrm = np.sqrt(np.einsum("cijk,cijk->ijk", y, y))[mask]
        drift = float(np.max(np.abs(nrm / mat.Ms[mask] - 1.0))) if nrm.size else 0.0
        if not np.isfinite(drift) or drift > BLOWUP_DRIFT:
            raise OracleBlowup(res.step + 1, res.t + dt, drift)
        res.m = renormalize(y, mat)
        k += 1
        res.t = t0 + k * dt
        res.step = step0 + k
        cur = mean_normalized(res.m, mat)
        res.final_residual = float(np.max(np.abs(cur - prev)))
        hit_eq = eq_tol is not None and res.final_residual < eq_tol
        prev = cur
        if hit_eq:
            reason = "equilibrated"
        if k % sample_every == 0 or k == n_total or hit_eq:
            res.rows.append(row(res.m, res.t))
        if hit_eq:
            break
    if not hit_eq and eq_tol is not None and k == n_total:
        reason = "not_converged"
    res.stop_reason = reason
    return res


# ----------------------------------------------------------------------------
# benchmark helpers (bench/common.py:40-48, bench/std4.py)
# ----------------------------------------------------------------------------

def stable_dt(dx, A, Ms, safety=0.5):
    """bench/common.py:40-48."""
    return safety * 2.5e-14 * (dx / 0.78125e-9) ** 2 * ((1.3e-11 / 8e5) / (A / Ms))


def timed_rk4_steps(m0, mat: Mat, terms: Terms, dt: float, nsteps: int):
    """Wall time of ``nsteps`` oracle RK4 steps (used as the CPU baseline)."""
    t0 = time.perf_counter()
    r = run(m0, mat, terms, "rk4", dt, max_steps=nsteps)
    return time.perf_counter() - t0, r
