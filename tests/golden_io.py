"""Helpers to load the golden fixtures made by tests/golden/make_golden.py."""
import glob
import os

import numpy as np

from oracle import magnex_oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLD, "*.npz"))
               if not os.path.basename(p).startswith(("tensor_known", "sp4_trace", "fno_")))


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
