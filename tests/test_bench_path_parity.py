"""The benchmarked demag path pinned against the CPU oracle directly.

The 512^3 bench runs the warp-FFT plane pipeline (yz_pipe.cu, L = 1024) and
the warp x passes (x_warp.cu, nx = 512) on the GPU-built mirrored tensor.
Here each of those kernels is compared with the oracle's convolution
(oracle.magnex_oracle.demag_field, a restatement of reference demag.py:203-216)
on the *same* spectra, read back from the device, so the only difference left
is FFT round-off; and the complex-spectra pipeline (kernel mode 5) is compared
with the oracle on the reference's own packed tensor (demag.py:183-195).

Tolerances: ||dH||_inf / ||H||_inf.  The FFT-only comparisons are held to
1e-13 (observed values are printed).  The tensor comparisons (GPU-built
tensor vs the reference tensor) are pinned at measured values: the reference
tensor is the difference of large Newell antiderivatives and changes at the
1e-10..1e-9 level when a single libm result moves by one ulp
(tests/test_tensor_noise_floor.py), so those bounds describe the reference's
own reproducibility, not FFT accuracy.  DESIGN.md section 6 records them.
"""
import os

import numpy as np
import pytest

import paper_2602_12242_b200 as mx
from oracle import magnex_oracle as O

pytestmark = pytest.mark.gpu


def nrm(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


class env:
    def __init__(self, **kv):
        self.kv = kv

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kv}
        os.environ.update({k: str(v) for k, v in self.kv.items()})

    def __exit__(self, *a):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def test_warp_pipeline_l1024_matches_oracle_on_its_spectra():
    """The bench's y/z kernel (k_yz_pipe_w, L = 1024, kernel mode 3) vs the
    oracle's scipy convolution with the spectra the device holds."""
    g = mx.GridSpec(16, 512, 512, 4e-9, 4e-9, 4e-9)
    k = mx.DemagKernel.build(g, symmetric=True)
    assert k.kmode == 3
    m = np.random.default_rng(21).standard_normal((3,) + g.shape) * 8e5
    h = k.field(m)
    ref = O.demag_field(k.spectra, m, workers=8)
    e = nrm(h, ref)
    print(f"L=1024 warp pipeline vs oracle (same spectra): {e:.3e}")
    assert e <= 1e-13


@pytest.mark.parametrize("pipe", ["1", "0"])
def test_warp_x_passes_nx512_match_oracle(pipe):
    """The bench's x passes (x_warp.cu, nx = 512): plane-major output for the
    pipeline (MXB_PIPE=1) and row-major for the 5-pass path."""
    g = mx.GridSpec(512, 16, 16, 4e-9, 4e-9, 4e-9)
    with env(MXB_PIPE=pipe):
        k = mx.DemagKernel.build(g, symmetric=True)
    assert k.pipeline == (pipe == "1")
    m = np.random.default_rng(22).standard_normal((3,) + g.shape) * 8e5
    h = k.field(m)
    ref = O.demag_field(k.spectra, m, workers=8)
    e = nrm(h, ref)
    print(f"nx=512 warp x passes (MXB_PIPE={pipe}) vs oracle: {e:.3e}")
    assert e <= 1e-13


@pytest.mark.parametrize("dims", [(8, 512, 512), (8, 256, 256)])
def test_complex_pipeline_on_reference_tensor(dims):
    """from_packed with the reference's packed tensor selects the plane
    pipeline with complex spectra (kernel mode 5); field vs the oracle."""
    cell = (2e-9, 2.5e-9, 3e-9)
    g = mx.GridSpec(*dims, *cell)
    packed = O.packed_tensor(*dims, *cell)
    k = mx.DemagKernel.from_packed(g, packed)
    assert k.kmode == 5 and k.pipeline
    m = np.random.default_rng(23).standard_normal((3,) + g.shape) * 8e5
    h = k.field(m)
    spec = O.kernel_spectra(packed, workers=8)
    del packed
    ref = O.demag_field(spec, m, workers=8)
    e = nrm(h, ref)
    print(f"complex pipeline {dims} vs oracle on the reference tensor: {e:.3e}")
    assert e <= 1e-13
    # the unfolded device spectra are the reference's
    assert nrm(k.spectra, spec) <= 1e-13
    # the 5-pass complex path agrees
    with env(MXB_PIPE="0"):
        k5 = mx.DemagKernel.from_packed(g, O.packed_tensor(*dims, *cell))
    assert k5.kmode == 0
    assert nrm(k5.field(m), h) <= 1e-13


def test_complex_pipeline_rk4_run_matches_oracle():
    """A graph-captured RK4 run through Simulation.run_until with the
    reference tensor in the complex-spectra pipeline, vs the oracle."""
    dims, cell = (8, 256, 256), (3e-9, 3e-9, 3e-9)
    g = mx.GridSpec(*dims, *cell)
    packed = O.packed_tensor(*dims, *cell)
    k = mx.DemagKernel.from_packed(g, packed)
    assert k.kmode == 5
    mat = mx.MaterialMap(g, Ms=8e5, A=1.3e-11, Ku=5e4, eK=(0, 0, 1), alpha=0.1)
    rhs = mx.PartitionedRHS(mat, exchange=True, anisotropy=True, demag=k, bias=(1e4, 0.0, 0.0))
    m0 = np.random.default_rng(24).standard_normal((3,) + g.shape)
    omat = O.make_mat(dims, cell, 8e5, A=1.3e-11, Ku=5e4, eK=(0, 0, 1), alpha=0.1)
    m0 = O.renormalize(m0, omat)
    st = mx.SimState(mx.VectorField3(g, m0.copy()))
    mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", 5e-14), sample_every=10 ** 9,
                  energy_in_samples=False).run_until(mx.StopCondition(max_steps=3))
    terms = O.Terms(exchange=True, anisotropy=True, spectra=O.kernel_spectra(packed, workers=8),
                    bias=np.array([1e4, 0.0, 0.0]))
    r = O.run(m0, omat, terms, "rk4", 5e-14, max_steps=3)
    e = float(np.max(np.abs(st.m.data - r.m)) / 8e5)
    print(f"3 RK4 steps, complex pipeline vs oracle: {e:.3e}")
    assert e <= 1e-12


# The GPU-built tensor (correctly rounded atan/asinh, dd_math.cuh) against the
# reference tensor, random-direction m (the bench's state), measured on B200
# (round 2): H_demag mirrored / unmirrored build and H_eff of the bench material
#   32^3   3.3e-11 / 1.5e-11   H_eff 1.4e-12
#   64^3   6.3e-10 / 3.7e-10   H_eff 2.8e-11
#   128^3  4.3e-9  / 2.3e-9    H_eff 2.0e-10
# (CUDA's asinh/atan gave 4.7e-10 / 1.1e-8 / 5.4e-8).  What is left is numpy's
# own misrounding (0.4% of arctan, 0.03% of arcsinh arguments) plus, for the
# mirrored build, the reference's asymmetric summation order: the reference's
# field itself moves by 4.0e-10 (32^3) and 8.6e-9 (64^3) between an AVX-512
# host and a glibc host (tests/test_tensor_noise_floor.py).  Pinned at about 2x.
SYM_DEV = {32: (7e-11, 3e-11, 3e-12), 64: (1.3e-9, 8e-10, 6e-11), 128: (9e-9, 5e-9, 4e-10)}


@pytest.mark.parametrize("n", [32, 64, 128])
def test_gpu_built_tensor_deviation_from_reference(n):
    cell = (4e-9, 4e-9, 4e-9)   # the bench's cell
    g = mx.GridSpec(n, n, n, *cell)
    packed = O.packed_tensor(n, n, n, *cell)
    spec = O.kernel_spectra(packed, workers=8)
    del packed
    rng = np.random.default_rng(25)
    m = rng.standard_normal((3,) + g.shape)
    m *= 8e5 / np.sqrt((m * m).sum(axis=0))
    ref = O.demag_field(spec, m, workers=8)
    ks = mx.DemagKernel.build(g, symmetric=True)
    ku = mx.DemagKernel.build(g)
    es, eu = nrm(ks.field(m), ref), nrm(ku.field(m), ref)
    # H_eff of the bench material (the north-star contract is on H_eff)
    mat = mx.MaterialMap(g, Ms=8e5, A=1.3e-11, Ku=5e4, eK=(0.0, 0.0, 1.0), D=1e-3, alpha=0.1)
    omat = O.make_mat((n, n, n), cell, 8e5, A=1.3e-11, Ku=5e4, eK=(0.0, 0.0, 1.0), D=1e-3, alpha=0.1)
    bias = np.array([1e4, 0.0, 0.0])
    terms = O.Terms(exchange=True, anisotropy=True, dmi=True, spectra=spec, bias=bias)
    href = O.h_eff(0.0, m, omat, terms)
    rhs = mx.PartitionedRHS(mat, exchange=True, anisotropy=True, dmi=True, demag=ks, bias=bias)
    eh = nrm(rhs.h_total_quiet(0.0, m), href)
    print(f"{n}^3: H_demag mirrored build {es:.3e}, unmirrored build {eu:.3e}; "
          f"H_eff (bench material, mirrored) {eh:.3e}")
    ds, du, dh = SYM_DEV[n]
    assert es <= ds and eu <= du and eh <= dh
    if n <= 64:
        assert eh <= 1e-10   # the north-star contract, on H_eff
