"""Warp-FFT x passes (x_warp.cu, nx = 512) against the radix-16 x passes and
the oracle, in the row-major (5-pass) and plane-major (pipeline) layouts."""
import os

import numpy as np
import pytest

import paper_2602_12242_b200 as mx
from oracle import magnex_oracle as O

pytestmark = pytest.mark.gpu


def field(g, m, xwarp, pipe, symmetric=True):
    env = {"MXB_XWARP": "1" if xwarp else "0", "MXB_PIPE": "1" if pipe else "0"}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        k = mx.DemagKernel.build(g, symmetric=symmetric)
        return k.field(m)
    finally:
        for key, v in old.items():
            if v is None:
                os.environ.pop(key, None)
            else:
                os.environ[key] = v


@pytest.mark.parametrize("dims,pipe", [((512, 16, 16), False), ((512, 8, 4), False), ((512, 64, 64), True),
                                       ((512, 16, 16), True)])
def test_warp_x_passes_match_radix16(dims, pipe):
    g = mx.GridSpec(*dims, 2e-9, 2.5e-9, 3e-9)
    m = np.random.default_rng(21).normal(size=(3,) + g.shape) * 8e5
    hw = field(g, m, True, pipe)
    h16 = field(g, m, False, pipe)
    assert np.linalg.norm(hw - h16) <= 1e-14 * np.linalg.norm(h16)


def test_warp_x_passes_match_oracle():
    dims, cell = (512, 2, 2), (2e-9, 2.5e-9, 3e-9)
    g = mx.GridSpec(*dims, *cell)
    packed = O.packed_tensor(*dims, *cell)
    k = mx.DemagKernel.from_packed(g, packed)
    m = np.random.default_rng(22).normal(size=(3,) + g.shape) * 8e5
    ref = O.demag_field(O.kernel_spectra(packed), m)
    assert np.max(np.abs(k.field(m) - ref)) <= 1e-12 * np.max(np.abs(ref))
