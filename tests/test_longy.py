"""Long y lines (py = 2048 / 4096, longy.cu): the plane-major row kernels and
the ky-contiguous fused z pass against the 5-pass column kernels
(MXB_LONGY=0) and the oracle.

Tolerances: against the 5-pass path on the same spectra <= 1e-13 normwise
(same radix-16 core, other pass order); against the oracle <= 1e-8 (the GPU
tensor builder's round-off, as in test_gpu_parity); the
spectra read back from either layout are bit-identical (same real parts)."""
import os

import numpy as np
import pytest

import paper_2602_12242_b200 as mx
from oracle import magnex_oracle as O

pytestmark = pytest.mark.gpu


def with_env(env, fn):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def nrm(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


def build(g, on):
    return with_env({"MXB_LONGY": "1" if on else "0"}, lambda: mx.DemagKernel.build(g, symmetric=True))


@pytest.mark.parametrize("dims", [(8, 1024, 4), (8, 2048, 8), (16, 2048, 16), (4, 1024, 64)])
def test_longy_matches_five_pass(dims):
    g = mx.GridSpec(*dims, 2e-9, 2.5e-9, 3e-9)
    m = np.random.default_rng(5).normal(size=(3,) + g.shape) * 8e5
    kl, k5 = build(g, True), build(g, False)
    assert nrm(kl.field(m), k5.field(m)) <= 1e-13


def test_longy_matches_oracle():
    dims, cell = (4, 1024, 2), (2e-9, 2.5e-9, 3e-9)
    g = mx.GridSpec(*dims, *cell)
    packed = O.packed_tensor(*dims, *cell)
    m = np.random.default_rng(6).normal(size=(3,) + g.shape) * 8e5
    ref = O.demag_field(O.kernel_spectra(packed), m)
    k = build(g, True)   # GPU tensor, mirrored octant: round-off from the reference tensor
    assert nrm(k.field(m), ref) <= 1e-8


def test_longy_spectra_readback():
    g = mx.GridSpec(4, 1024, 4, 2e-9, 2e-9, 2e-9)
    assert np.array_equal(build(g, True).spectra, build(g, False).spectra)


def test_longy_rk4_run():
    g = mx.GridSpec(8, 1024, 4, 4e-9, 4e-9, 4e-9)
    mat = mx.MaterialMap(g, Ms=8e5, A=1.3e-11, alpha=0.02)
    m0 = np.zeros((3,) + g.shape)
    m0[0] = 1.0
    m0 += 0.05 * np.random.default_rng(8).normal(size=m0.shape)
    m0 = mx.VectorField3(g, m0)
    mx.renormalize(m0, mat)

    def run(on):
        rhs = mx.PartitionedRHS(mat, exchange=True, demag=build(g, on), bias=(1e4, 0, 0))
        st = mx.SimState(m0.copy())
        sim = mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", 1e-13), sample_every=1, energy_in_samples=False)
        tr = sim.run_until(mx.StopCondition(max_steps=5))
        return st.m.data, np.stack([tr.column(c) for c in ("mx", "my", "mz")], 1)

    ml, tl = run(True)
    m5, t5 = run(False)
    assert nrm(ml, m5) <= 1e-12
    assert np.max(np.abs(tl - t5)) <= 1e-12
