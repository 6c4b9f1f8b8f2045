"""Seeded FNO tensor tables shared by the golden generator and the tests
(same construction as tests/golden/make_golden_fno.py; pinned by SHA-256)."""
import hashlib
import os

import numpy as np

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FNO_CASES = ("small_gelu", "small_relu", "film_w32")


def tensors(width, modes, seed, scale=0.2):
    rng = np.random.default_rng(seed)
    m1, m2 = modes
    r = lambda *s: (rng.standard_normal(s) * scale).astype(np.float32)  # noqa: E731
    c = lambda *s: ((rng.standard_normal(s) + 1j * rng.standard_normal(s)) * 0.1 / np.sqrt(width)).astype(np.complex64)  # noqa: E731
    t = {"lift.weight": r(width, 3), "lift.bias": r(width)}
    for k in range(4):
        t[f"block{k}.spectral.pos"] = c(width, width, m1, m2)
        t[f"block{k}.spectral.neg"] = c(width, width, m1, m2)
        t[f"block{k}.local.weight"] = (rng.standard_normal((width, width)) / np.sqrt(width)).astype(np.float32)
        t[f"block{k}.local.bias"] = r(width)
    t["proj.weight"] = r(3, width)
    t["proj.bias"] = r(3)
    t["norm.in_mean"] = np.array([0.1, -0.2, 0.05], np.float32)
    t["norm.in_std"] = np.array([0.9, 1.1, 0.7], np.float32)
    t["norm.out_mean"] = np.array([1e3, -2e3, 5e2], np.float32)
    t["norm.out_std"] = np.array([3e4, 2e4, 4e4], np.float32)
    return t


def table_sha(t):
    h = hashlib.sha256()
    for k in sorted(t):
        h.update(k.encode())
        h.update(np.ascontiguousarray(t[k]).tobytes())
    return h.hexdigest()


def load_case(name):
    z = dict(np.load(os.path.join(GOLD, f"fno_{name}.npz")))
    t = tensors(int(z["width"]), (int(z["m1"]), int(z["m2"])), int(z["seed"]))
    assert table_sha(t) == str(z["table_sha"]), "seeded tensor table drifted from the golden"
    return t, z
