"""Golden vectors for the FNO surrogate, produced by the reference itself.

Run in the build container (the reference is importable there, not on the GPU
box):  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_fno.py
Writes tests/golden/fno_*.npz: the f32/c64 tensor table, inputs, and the
reference outputs of FnoModel.infer and spectral_conv (magnex/fno.py).
"""
import os
import sys

import numpy as np

from magnex import fno as F  # noqa: E402  (reference package)

HERE = os.path.dirname(os.path.abspath(__file__))


def tensors(width, modes, seed, scale=0.2):
    """Seeded tensor table (also rebuilt by tests/fno_tables.py; pinned by SHA-256)."""
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
    import hashlib
    h = hashlib.sha256()
    for k in sorted(t):
        h.update(k.encode())
        h.update(np.ascontiguousarray(t[k]).tobytes())
    return h.hexdigest()


def case(name, width, modes, H, W, seed, activation, with_sc=True):
    t = tensors(width, modes, seed)
    model = F.FnoModel.from_tensors(t, activation=activation)
    rng = np.random.default_rng(seed + 100)
    x = rng.standard_normal((3, H, W))
    y = model.infer(x)
    out = dict(x=x, y=y, activation=activation, width=width, m1=modes[0], m2=modes[1], seed=seed,
               table_sha=table_sha(t))
    if with_sc:
        v = rng.standard_normal((width, H, W))
        out.update(v=v, sc=F.spectral_conv(v, model.spec_pos[0], model.spec_neg[0]))
    np.savez_compressed(os.path.join(HERE, f"fno_{name}.npz"), **out)
    print(name, x.shape, float(np.max(np.abs(y))))


if __name__ == "__main__":
    sys.path.insert(0, HERE)
    case("small_gelu", 4, (3, 3), 8, 10, 21, F.ACT_GELU)
    case("small_relu", 4, (3, 2), 12, 10, 22, F.ACT_RELU)
    case("film_w32", 32, (12, 12), 32, 128, 23, F.ACT_GELU, with_sc=False)
