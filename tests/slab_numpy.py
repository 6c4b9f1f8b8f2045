"""Numpy slab backend for the gloo tests of paper_2602_12242_b200.slab -- TEST
INFRASTRUCTURE.  It implements the same per-rank operations as
CudaSlabBackend (demag x-forward into per-destination kx chunks, y/z on the
kx chunk, x-inverse; the fused stage with halo planes; step partials and
commit) on top of the CPU oracle, so SlabSimulation's orchestration runs
unchanged under torch.distributed/gloo on CPU."""
from __future__ import annotations

import numpy as np
import torch

from oracle import magnex_oracle as O
from paper_2602_12242_b200 import _lib as L


class Stats:
    def __init__(self):
        self.steps_done = 0
        self.status = 0
        self.mean = np.zeros(3)
        self.residual = float("nan")
        self.drift = 0.0
        self.dead_flat = -1


class NumpySlabBackend:
    def __init__(self, plan, mat_global: O.Mat, spectra_global, terms: L.Terms):
        self.torch = torch
        self.plan = plan
        z0, nzl = plan.z0, plan.nz_local
        self.matg = mat_global
        self.mat = self._slice_mat(z0, z0 + nzl)
        shape = (3, nzl, plan.ny, plan.nx)
        self.fields = {k: torch.zeros(shape, dtype=torch.float64)
                       for k in ("Y0", "Y1", "P", "K1", "S", "HD")}
        self.halo = {k: torch.zeros((3, plan.ny, plan.nx), dtype=torch.float64)
                     for k in ("send_lo", "send_hi", "lo", "hi")}
        n = 2 * plan.nranks * plan.block_elems
        self.send = torch.zeros(n, dtype=torch.float64)
        # one rank: no exchange, both sides of the transpose are the same buffer
        self.recv = self.send if plan.nranks == 1 else torch.zeros(n, dtype=torch.float64)
        self.spectra = spectra_global
        self.ctl = Stats()
        self._red = torch.zeros(8, dtype=torch.float64)
        self.prev = np.zeros(3)
        self.n_mag = 1
        self.eq_tol = -1.0

    def _slice_mat(self, za, zb):
        m = self.matg
        sl = (lambda a: None if a is None else a[za:zb])  # noqa: E731
        return O.Mat((m.dims[0], m.dims[1], zb - za), m.cell, m.Ms[za:zb], m.A[za:zb], m.Ku[za:zb],
                     m.D[za:zb], m.alpha[za:zb], m.eK[:, za:zb], m.gamma, sl(m.Kc1), m.c1, m.c2,
                     sl(m.Db))

    # -- data movement -----------------------------------------------------------
    def upload(self, name, host):
        self.fields[name].copy_(torch.from_numpy(np.ascontiguousarray(host)))

    def download(self, name):
        return self.fields[name].numpy().copy()

    def boundary_planes(self, name):
        f = self.fields[name]
        self.halo["send_lo"].copy_(f[:, 0])
        self.halo["send_hi"].copy_(f[:, -1])
        return self.halo["send_lo"], self.halo["send_hi"], self.halo["lo"], self.halo["hi"]

    def new_tensor(self, host):
        return torch.as_tensor(np.asarray(host, dtype=np.float64))

    # -- demag ----------------------------------------------------------------------
    def _blocks(self, t):
        p = self.plan
        return t.numpy().view(np.complex128).reshape(p.nranks, p.nz_local, p.ny, p.chunk_pitch, 3)

    def demag_x_forward(self, src):
        p = self.plan
        px = 2 * p.nx if p.nx > 1 else 1
        X = np.fft.rfft(self.fields[src].numpy(), n=px, axis=-1)   # (3, nzl, ny, hx)
        S = self._blocks(self.send)
        S[...] = 0
        for kx in range(p.hx):
            b, kc = divmod(kx, p.chunk)
            S[b, :, :, kc, :] = np.moveaxis(X[:, :, :, kx], 0, -1)

    def demag_yz(self):
        p = self.plan
        pz = 2 * p.nz if p.nz > 1 else 1
        py = 2 * p.ny if p.ny > 1 else 1
        Rb = self._blocks(self.recv).reshape(p.nz, p.ny, p.chunk_pitch, 3)
        kn = p.kx_count
        A = np.moveaxis(Rb[:, :, :kn, :], -1, 0)                   # (3, nz, ny, kn)
        F = np.fft.fft(np.fft.fft(A, n=py, axis=2), n=pz, axis=1)
        K = self.spectra[:, :, :, p.kx0:p.kx0 + kn]
        H = np.empty_like(F)
        for a, mix in enumerate(O.MIX):
            H[a] = K[mix[0]] * F[0] + K[mix[1]] * F[1] + K[mix[2]] * F[2]
        Hb = np.fft.ifft(np.fft.ifft(H, axis=1)[:, :p.nz], axis=2)[:, :, :p.ny]
        Rb[:, :, :kn, :] = np.moveaxis(Hb, 0, -1)

    def demag_x_inverse(self, dst):
        p = self.plan
        px = 2 * p.nx if p.nx > 1 else 1
        S = self._blocks(self.send)
        X = np.empty((3, p.nz_local, p.ny, p.hx), dtype=np.complex128)
        for kx in range(p.hx):
            b, kc = divmod(kx, p.chunk)
            X[:, :, :, kx] = np.moveaxis(S[b, :, :, kc, :], -1, 0)
        self.fields[dst].copy_(torch.from_numpy(np.fft.irfft(X, n=px, axis=-1)[..., :p.nx].copy()))

    # -- stencil stage ----------------------------------------------------------------
    def stage(self, mode, terms: L.Terms, *, ys, y, out, hd=None, k1=None, s=None, k1_out=None,
              halo_lo=False, halo_hi=False, bias=(0.0, 0.0, 0.0), c=0.0, dt6=0.0, renorm=True):
        p = self.plan
        if self.ctl.status:
            return   # halted: the device stage kernels are no-ops too
        f = {k: v.numpy() for k, v in self.fields.items()}
        m = f[ys]
        parts = ([self.halo["lo"].numpy()[:, None]] if halo_lo else []) + [m] + \
            ([self.halo["hi"].numpy()[:, None]] if halo_hi else [])
        ext = np.concatenate(parts, axis=1)
        za = p.z0 - (1 if halo_lo else 0)
        matx = self._slice_mat(za, za + ext.shape[1])
        mask = terms.mask
        ghost = {0: "neumann", 1: "dmi", 2: "periodic"}[terms.ghost_mode]
        tl = O.Terms(exchange=bool(mask & L.TERM_EXCHANGE), anisotropy=bool(mask & L.TERM_ANISOTROPY),
                     dmi=bool(mask & L.TERM_DMI), ghost_mode=ghost, cubic=bool(mask & L.TERM_CUBIC),
                     bulk_dmi=bool(mask & L.TERM_BULK_DMI))
        h = O.h_eff(0.0, ext, matx, tl)
        lo = 1 if halo_lo else 0
        h = h[:, lo:lo + p.nz_local]
        if mask & L.TERM_DEMAG:
            h = h + f[hd]
        if mask & L.TERM_BIAS:
            h = h + np.asarray(bias).reshape(3, 1, 1, 1)
        k = O.llg_rhs(m, h, self.mat, bool(terms.precession), bool(terms.damping))
        if mode == 0:
            f[out][...] = h
            return
        if mode == 1:
            f[out][...] = k
            return
        yv = f[y]
        if mode in (2, 3, 4, 6):
            v = yv + c * k
            if mode == 2:
                f[k1_out][...] = k
            elif mode == 3:
                f[s][...] = k
            elif mode == 4:
                f[s][...] = f[s] + k
        else:
            v = yv + dt6 * (f[k1] + 2.0 * f[s] + k)
        if mode in (5, 6):
            mk = self.mat.mask
            nr = np.sqrt(np.einsum("cijk,cijk->ijk", v, v))[mk]
            drift = float(np.max(np.abs(nr / self.mat.Ms[mk] - 1.0))) if nr.size else 0.0
            v = O.renormalize(v, self.mat)
            with np.errstate(invalid="ignore", divide="ignore"):
                q = v / np.where(mk, self.mat.Ms, 1.0)
            sums = [q[cc][mk].sum() for cc in range(3)]
            self._red[:] = torch.tensor([*sums, 0.0, drift, float(self.ctl.status), -9e18, 0.0])
        elif renorm:
            v = O.renormalize(v, self.mat)
        f[out][...] = v

    def partials(self):
        return self._red

    def commit(self, totals):
        t = totals.numpy()
        c = self.ctl
        if c.status:
            return
        drift = t[4]
        if not np.isfinite(drift) or drift > 0.10:
            c.status, c.drift = L.EBLOWUP, drift
            return
        mean = t[:3] / self.n_mag
        c.residual = float(np.max(np.abs(mean - self.prev)))
        c.mean = mean
        self.prev = mean
        c.drift = drift
        c.steps_done += 1
        if self.eq_tol >= 0 and c.residual < self.eq_tol:
            c.status = L.EQUILIBRATED

    def ctl_reset(self, prev_mean, n_magnetic, eq_tol):
        self.ctl = Stats()
        self.prev = np.asarray(prev_mean, dtype=np.float64)
        self.ctl.mean = self.prev.copy()
        self.n_mag = n_magnetic
        self.eq_tol = eq_tol

    def ctl_get(self):
        return self.ctl

    def local_mean_sums(self, name):
        m = self.download(name)
        mk = self.mat.mask
        with np.errstate(invalid="ignore", divide="ignore"):
            q = m / np.where(mk, self.mat.Ms, 1.0)
        return np.array([q[cc][mk].sum() for cc in range(3)]), int(np.count_nonzero(mk))
