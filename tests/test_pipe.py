"""The L2-resident y/z plane pipeline (yz_pipe.cu, kmode 3) against the
5-pass path it replaces: same FFT code and twiddles, so the fields must be
bit-identical; also the unfolded spectra and a graph-captured RK4 run."""
import os

import numpy as np
import pytest

import paper_2602_12242_b200 as mx
from paper_2602_12242_b200 import _lib as L

pytestmark = pytest.mark.gpu


def build(g, pipe):
    old = os.environ.get("MXB_PIPE")
    os.environ["MXB_PIPE"] = "1" if pipe else "0"
    try:
        return mx.DemagKernel.build(g, symmetric=True)
    finally:
        if old is None:
            del os.environ["MXB_PIPE"]
        else:
            os.environ["MXB_PIPE"] = old


@pytest.mark.parametrize("dims", [(8, 8, 8), (16, 16, 16), (64, 32, 32), (8, 64, 64), (32, 128, 128)])
def test_pipeline_matches_five_pass_bitwise(dims):
    g = mx.GridSpec(*dims, 2e-9, 2.5e-9, 3e-9)
    kp, k5 = build(g, True), build(g, False)
    m = np.random.default_rng(11).normal(size=(3,) + g.shape) * 8e5
    hp, h5 = kp.field(m), k5.field(m)
    assert np.array_equal(hp, h5), np.max(np.abs(hp - h5)) / np.max(np.abs(h5))
    # repeated evaluations reuse the slots and barrier counter
    assert np.array_equal(kp.field(m), hp)
    assert np.array_equal(kp.spectra, k5.spectra)


def test_pipeline_refuses_generic_switch():
    g = mx.GridSpec(16, 16, 16, 2e-9, 2e-9, 2e-9)
    kp = build(g, True)
    with pytest.raises(ValueError, match="plane pipeline"):
        kp.set_fast(False)


def test_pipeline_rk4_run_bitwise():
    g = mx.GridSpec(32, 32, 32, 3e-9, 3e-9, 3e-9)
    mat = mx.MaterialMap(g, Ms=8e5, A=1.3e-11, Ku=5e4, eK=(0, 0, 1), alpha=0.1)
    m0 = mx.VectorField3(g, np.random.default_rng(3).normal(size=(3,) + g.shape))
    mx.renormalize(m0, mat)
    out = []
    for pipe in (True, False):
        rhs = mx.PartitionedRHS(mat, exchange=True, anisotropy=True, demag=build(g, pipe),
                                bias=(1e4, 0.0, 0.0))
        st = mx.SimState(m0.copy())
        mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", 5e-14), sample_every=10 ** 9,
                      energy_in_samples=False).run_until(mx.StopCondition(max_steps=6))
        out.append(st.m.data.copy())
    assert np.array_equal(out[0], out[1])


def test_warp_fft_pipeline_matches_five_pass():
    """Opt-in warp-per-line FFT variant (fft_warp.cuh, L = 1024): different
    rounding from the radix-16 path, so a normwise tolerance."""
    g = mx.GridSpec(8, 512, 512, 2e-9, 2.5e-9, 3e-9)
    m = np.random.default_rng(12).normal(size=(3,) + g.shape) * 8e5
    h5 = build(g, False).field(m)
    old = os.environ.get("MXB_PIPE_WARP")
    os.environ["MXB_PIPE_WARP"] = "1"
    try:
        hw = build(g, True).field(m)
    finally:
        if old is None:
            del os.environ["MXB_PIPE_WARP"]
        else:
            os.environ["MXB_PIPE_WARP"] = old
    assert np.linalg.norm(hw - h5) <= 1e-13 * np.linalg.norm(h5)


@pytest.mark.parametrize("dims", [(64, 256, 256), (8, 256, 256)])
def test_warp_pair_pipeline_l512_matches_five_pass(dims):
    """Warp pipeline with two 512-point lines per warp (k_yz_pipe_w512)."""
    g = mx.GridSpec(*dims, 2e-9, 2.5e-9, 3e-9)
    m = np.random.default_rng(13).normal(size=(3,) + g.shape) * 8e5
    hp, h5 = build(g, True).field(m), build(g, False).field(m)
    assert np.linalg.norm(hp - h5) <= 1e-13 * np.linalg.norm(h5)


def test_warp_pipeline_in_graph_captured_run():
    """RK4 through Simulation.run_until (mxb_run replays captured CUDA graphs,
    the slot tensor map travels as a kernel parameter) with the warp-FFT
    plane pipeline at L = 1024, against the 5-pass path."""
    g = mx.GridSpec(16, 512, 512, 3e-9, 3e-9, 3e-9)
    mat = mx.MaterialMap(g, Ms=8e5, A=1.3e-11, Ku=5e4, eK=(0, 0, 1), alpha=0.1)
    m0 = mx.VectorField3(g, np.random.default_rng(4).normal(size=(3,) + g.shape))
    mx.renormalize(m0, mat)
    out = []
    for pipe in (True, False):
        k = build(g, pipe)
        assert k.pipeline == pipe
        rhs = mx.PartitionedRHS(mat, exchange=True, anisotropy=True, demag=k, bias=(1e4, 0.0, 0.0))
        st = mx.SimState(m0.copy())
        mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", 5e-14), sample_every=10 ** 9,
                      energy_in_samples=False).run_until(mx.StopCondition(max_steps=4))
        out.append(st.m.data.copy())
    assert np.max(np.abs(out[0] - out[1])) <= 1e-12 * 8e5
