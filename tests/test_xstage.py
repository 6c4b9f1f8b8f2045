"""The x-row fused stage (stencil.cu k_stage_x, opt-in MXB_XFUSE=1: x c2r of
the demag spectra -> stage update -> x r2c of the new state, one kernel per
RK4 stage) against the unfused kernels it replaces (k_c2r_w, k_stage_zt,
k_r2c_w; the default path).

Same arithmetic in the same order as the TMA z-march stage kernel, so the
state after a run is bit-identical where the unfused path runs that kernel;
the <m> samples differ only in the order the per-block partial sums are
added (the fused kernel reduces per row pair, the z-march per 32 x 4 x 64
tile): <= 1e-15 relative.  The unfused path is itself pinned against the
oracle (test_gpu_parity.py, test_bench_path_parity.py).
"""
import ctypes as C
import os

import numpy as np
import pytest

import paper_2602_12242_b200 as mx
from paper_2602_12242_b200 import _lib as L
from paper_2602_12242_b200.llg import _ORDER

pytestmark = pytest.mark.gpu

MS = 8e5


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


def pipe_kernel(g):
    k = with_env({"MXB_PIPE": "1"}, lambda: mx.DemagKernel.build(g, symmetric=True))
    assert k.pipeline
    return k


def run(g, mat, kern, m0, env, steps=3, bias=(1e4, 0.0, 0.0), dt=2e-14, sample_every=1,
        renorm=True, **terms):
    terms = terms or dict(exchange=True, anisotropy=True, dmi=True)
    rhs = mx.PartitionedRHS(mat, demag=kern, bias=bias, **terms)
    st = mx.SimState(mx.VectorField3(g, m0.copy()))
    sim = mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", dt, renorm_each_stage=renorm),
                        sample_every=sample_every, energy_in_samples=False)
    tr = with_env(env, lambda: sim.run_until(mx.StopCondition(max_steps=steps)))
    return st.m.data.copy(), np.stack([tr.column(c) for c in ("mx", "my", "mz")], 1)


def rand_m(g, seed):
    m = np.random.default_rng(seed).normal(size=(3,) + g.shape)
    return m * (MS / np.sqrt((m * m).sum(axis=0)))


def zt_grid(g):
    """The unfused path runs the TMA z-march stage kernel (heff_nb, the fused
    kernel's arithmetic) when its 32 x 4 x 64 tiles fill the GPU; smaller
    grids take the one-cell-per-thread kernel, whose exchange sum rounds
    differently (<= 1e-13, test_full_size.py)."""
    return -(-g.nx // 32) * -(-g.ny // 4) * -(-g.nz // 64) >= 4 * 148


def check_same(a, b, bitwise):
    (ma, ta), (mb, tb) = a, b
    if bitwise:
        assert np.array_equal(ma, mb), float(np.max(np.abs(ma - mb)) / MS)
        tol = 1e-15
    else:
        assert float(np.max(np.abs(ma - mb)) / MS) <= 1e-13
        tol = 1e-13
    assert ta.shape == tb.shape
    assert np.max(np.abs(ta - tb)) <= tol * max(1.0, float(np.max(np.abs(tb))))


MAT = dict(Ms=MS, A=1.3e-11, Ku=5e4, eK=(0.0, 0.0, 1.0), D=1e-3, alpha=0.1)


# (nx, ny, nz): the fused kernel takes nx = 512 x-rows; the plane pipeline ny = nz
@pytest.mark.parametrize("dims", [(512, 128, 128), (512, 16, 16), (512, 8, 8)], ids=["n128", "n16", "n8"])
def test_fused_stage_bitwise(dims):
    g = mx.GridSpec(*dims, 3e-9, 3e-9, 3e-9)
    mat = mx.MaterialMap(g, **MAT)
    kern = pipe_kernel(g)
    m0 = rand_m(g, 5)
    check_same(run(g, mat, kern, m0, {"MXB_XFUSE": "1"}), run(g, mat, kern, m0, {"MXB_XFUSE": "0"}), zt_grid(g))


def test_fused_stage_time_dependent_bias_and_no_stage_renorm():
    """A bias that changes per stage (host stage-bias path, no graph replay)
    and the stage states left unnormalised."""
    g = mx.GridSpec(512, 128, 128, 2e-9, 2.5e-9, 3e-9)
    mat = mx.MaterialMap(g, Ms=MS, A=1.3e-11, Ku=2e4, eK=(0.3, 0.0, 1.0), alpha=0.05)

    def bias(t):
        return (2e4 * np.cos(2e11 * t), 5e3, -1e4 * np.sin(3e11 * t))

    kern = pipe_kernel(g)
    m0 = rand_m(g, 6)
    kw = dict(bias=bias, renorm=False, exchange=True, anisotropy=True)
    check_same(run(g, mat, kern, m0, {"MXB_XFUSE": "1"}, **kw), run(g, mat, kern, m0, {"MXB_XFUSE": "0"}, **kw), zt_grid(g))


def test_fused_stage_spatial_bias_field():
    g = mx.GridSpec(512, 16, 16, 3e-9, 3e-9, 3e-9)
    mat = mx.MaterialMap(g, **MAT)
    field = np.random.default_rng(7).normal(size=(3,) + g.shape) * 1e4
    kern = pipe_kernel(g)
    m0 = rand_m(g, 8)
    kw = dict(bias=lambda t: field * (1.0 + 1e10 * t), exchange=True, dmi=True)
    check_same(run(g, mat, kern, m0, {"MXB_XFUSE": "1"}, **kw), run(g, mat, kern, m0, {"MXB_XFUSE": "0"}, **kw), zt_grid(g))


def test_fused_stage_exact_mode():
    """numpy-rounding stage arithmetic (MXB_EXACT / set_exact): the fused kernel's E=true instance."""
    g = mx.GridSpec(512, 128, 128, 3e-9, 3e-9, 3e-9)
    old = L.exact()
    L.set_exact(True)
    try:
        mat = mx.MaterialMap(g, **MAT)
        kern = pipe_kernel(g)
        m0 = rand_m(g, 9)
        check_same(run(g, mat, kern, m0, {"MXB_XFUSE": "1"}), run(g, mat, kern, m0, {"MXB_XFUSE": "0"}), zt_grid(g))
    finally:
        L.set_exact(old)


def test_fused_stage_is_the_path_taken():
    """mxb_time_steps reports the launches of the path it ran: 10 per step fused
    (x forward, 4 x (pipeline + fused stage), finalize), 17 unfused."""
    g = mx.GridSpec(512, 32, 32, 3e-9, 3e-9, 3e-9)
    mat = mx.MaterialMap(g, **MAT)
    kern = pipe_kernel(g)
    rhs = mx.PartitionedRHS(mat, exchange=True, anisotropy=True, dmi=True, demag=kern, bias=(1e4, 0, 0))
    ctx = mat._ctx()
    st = mx.VectorField3(g, rand_m(g, 10))
    L.check(ctx.call("mxb_state_set", L.dptr(np.ascontiguousarray(st.data))), "state")
    ts = rhs._terms_struct(tuple(x for x in _ORDER if x in rhs.enabled_terms()))
    bias = np.array([1e4, 0.0, 0.0])
    ms, nl = C.c_double(), C.c_int64()

    def launches(env):
        def f():
            L.check(ctx.call("mxb_time_steps", kern._d.h, C.byref(ts), 2e-14, 2, L.dptr(bias),
                             C.byref(ms), None, C.byref(nl)), "time_steps")
            return nl.value
        return with_env(env, f)

    assert launches({"MXB_XFUSE": "1"}) == 2 * 10
    assert launches({}) == 2 * 17
