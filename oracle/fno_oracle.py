"""CPU restatement of the reference FNO demag surrogate (TEST INFRASTRUCTURE ONLY).

Follows magnex/fno.py (pkg/src/magnex/fno.py) operation by operation so the
results are bit-identical to the reference on the same inputs:
  gelu / relu              fno.py:70-77
  spectral_conv            fno.py:228-255  (numpy.fft rfft2 / irfft2, einsum)
  normalizer               fno.py:187-213
  FnoModel.infer           fno.py:372-394
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline may import it.
"""
from __future__ import annotations

import numpy as np
from scipy.special import erf

N_BLOCKS = 4


def gelu(x):
    return 0.5 * x * (1 + erf(x / np.sqrt(2)))


def relu(x):
    return np.maximum(x, 0.0)


def spectral_conv(x, w_pos, w_neg):
    x = np.asarray(x, np.float64)
    c, H, W = x.shape
    ci, co, m1, m2 = w_pos.shape
    xf = np.fft.rfft2(x)
    out = np.zeros((co, H, W // 2 + 1), np.complex128)
    out[:, :m1, :m2] = np.einsum("ixy,ioxy->oxy", xf[:, :m1, :m2], w_pos)
    out[:, -m1:, :m2] = np.einsum("ixy,ioxy->oxy", xf[:, -m1:, :m2], w_neg)
    return np.fft.irfft2(out, s=(H, W))


def infer(t: dict, x, activation: int = 0):
    """Forward pass of the tensor table ``t`` (float64 / complex128 arrays) on (3,H,W)."""
    act = gelu if activation == 0 else relu
    x = np.ascontiguousarray(x, np.float64)
    im, isd = t["norm.in_mean"], t["norm.in_std"]
    om, osd = t["norm.out_mean"], t["norm.out_std"]
    xn = (x - im[:, None, None]) / isd[:, None, None]
    v = np.einsum("oc,chw->ohw", t["lift.weight"], xn) + t["lift.bias"][:, None, None]
    for k in range(N_BLOCKS):
        s = spectral_conv(v, t[f"block{k}.spectral.pos"], t[f"block{k}.spectral.neg"])
        local = (np.einsum("oc,chw->ohw", t[f"block{k}.local.weight"], v)
                 + t[f"block{k}.local.bias"][:, None, None])
        v = s + local
        if k < N_BLOCKS - 1:
            v = act(v)
    y = np.einsum("oc,chw->ohw", t["proj.weight"], v) + t["proj.bias"][:, None, None]
    return y * osd[:, None, None] + om[:, None, None]


def as_f64(tensors: dict) -> dict:
    """MAGW tensors (f32 / complex64) widened as the reference does (fno.py:300-322)."""
    return {k: (np.asarray(v, np.complex128) if np.iscomplexobj(v) else np.asarray(v, np.float64))
            for k, v in tensors.items()}
