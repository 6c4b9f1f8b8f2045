"""Helpers to load the golden fixtures made by tests/golden/make_golden.py."""
import glob
import os

import numpy as np

from oracle import magnex_oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLD, "*.npz"))
               if not os.path.basename(p).startswith(("tensor_known", "sp4_trace", "fno_", "spatial_bias", "bench_32",
                                                           "sp4_protocol")))


def load(name):
    return dict(np.load(os.path.join(GOLD, name + ".npz"), allow_pickle=False))


def mat_of(z):
    dims = tuple(int(v) for v in z["dims"])
    cell = tuple(float(v) for v in z["cell"])
    return O.Mat(dims, cell, z["Ms"], z["A"], z["Ku"], z["D"], z["alpha"], z["eK"])


def terms_of(z, spectra=None):
    t = set(str(s) for s in z["terms"])
    return O.Terms(exchange="exchange" in t, anisotropy="anisotropy" in t, dmi="dmi" in t,
                   spectra=spectra, bias=z["bias"] if bool(z["has_bias"]) else None,
                   ghost_mode=str(z["ghost_mode"]))


def packed_of(z):
    nx, ny, nz = (int(v) for v in z["dims"])
    dx, dy, dz = (float(v) for v in z["cell"])
    return O.packed_tensor(nx, ny, nz, dx, dy, dz)


class BiasReplay:
    """t -> the recorded (3,nz,ny,nx) bias field of the reference run at t
    (tests/golden/make_golden.py spatial_bias_golden): the reference's
    ScenarioConfig.build_bias callable, replayed bit for bit.  Stage times are
    matched to the nearest recorded time (|dt| <= 1e-9 of the step)."""

    def __init__(self, times, fields, dt):
        self.times = np.asarray(times)
        self.fields = fields
        self.tol = 1e-9 * dt

    def __call__(self, t):
        i = int(np.argmin(np.abs(self.times - t)))
        if abs(self.times[i] - t) > self.tol:
            raise KeyError(f"no recorded bias at t = {t!r}")
        return self.fields[i].copy()


def spatial_case(method):
    z = load("spatial_bias")
    Ms = z["Ms"]
    nz, ny, nx = Ms.shape
    mat = O.Mat((nx, ny, nz), (2e-9, 2e-9, 2e-9), Ms, z["A"], z["Ku"], np.zeros_like(Ms),
                z["alpha"], z["eK"])
    dt = float(z[method + "_dt"])
    return z, mat, dt, BiasReplay(z[method + "_times"], z[method + "_fields"], dt)
