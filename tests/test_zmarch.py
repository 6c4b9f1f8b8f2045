"""The z-marching stage kernels (stencil.cu: k_stage_zt with TMA-staged
planes, k_stage_zm with a shared-memory plane tile) at a grid large enough to
select them (>= 4 x 148 column tiles), against the oracle and against the
one-cell-per-thread kernel (MXB_ZMARCH=0) and the non-TMA z-march (MXB_ZTMA=0).

Tolerances: local terms in exact mode bit-identical to the oracle; H_eff,
rhs and one step <= 1e-12 normwise (contract 1e-10); the TMA and non-TMA
z-march compute the same expressions in the same order: bit-identical."""
import os

import numpy as np
import pytest

import paper_2602_12242_b200 as mx
from oracle import magnex_oracle as O

pytestmark = pytest.mark.gpu

DIMS, CELL = (512, 128, 64), (2e-9, 2e-9, 2e-9)


def nrm(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


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


@pytest.fixture(scope="module")
def case():
    g = mx.GridSpec(*DIMS, *CELL)
    kw = dict(Ms=8e5, A=1.3e-11, Ku=4e5, eK=(0.2, 0.1, 1.0), D=3e-3, alpha=0.3)
    mat = mx.MaterialMap(g, **kw)
    omat = O.make_mat(DIMS, CELL, **kw)
    m0 = np.random.default_rng(7).normal(size=(3,) + g.shape)
    m0 = O.renormalize(m0, omat)
    return g, mat, omat, m0


@pytest.fixture(params=[True, False], ids=["exact", "fast"])
def mode(request):
    mx.set_exact(request.param)
    yield request.param
    mx.set_exact(False)


@pytest.mark.parametrize("ztma", ["1", "0"])
def test_zmarch_heff_and_steps_match_oracle(case, mode, ztma):
    g, mat, omat, m0 = case
    bias = (1e4, -2e4, 3e4)
    rhs = mx.PartitionedRHS(mat, exchange=True, anisotropy=True, dmi=True, bias=bias)
    terms = O.Terms(exchange=True, anisotropy=True, dmi=True, bias=np.array(bias))
    plan = O.Plan(omat, terms.mode())
    f = lambda t, y: O.rhs_total(t, y, omat, terms, plan)
    env = {"MXB_ZTMA": ztma}
    h = with_env(env, lambda: rhs.h_total_quiet(0.0, m0))
    assert nrm(h, O.h_eff(0.0, m0, omat, terms, plan)) <= 1e-12
    r = with_env(env, lambda: rhs.rhs_total(0.0, m0))
    assert nrm(r, f(0.0, m0)) <= 1e-12
    dt = 2e-14
    post = lambda y: O.renormalize(y, omat)
    for method, ref in (("rk4", O.rk4_step(m0, 0.0, dt, f, post)), ("euler", O.euler_step(m0, 0.0, dt, f))):
        st = mx.SimState(mx.VectorField3(g, m0.copy()))
        sim = mx.Simulation(st, rhs, mx.IntegratorSpec(method, dt), energy_in_samples=False)
        with_env(env, lambda: sim.run_until(mx.StopCondition(max_steps=1)))
        assert nrm(st.m.data, O.renormalize(ref, omat)) <= 1e-12, method


@pytest.mark.parametrize("method", ["rk4", "euler"])
def test_tma_zmarch_is_bit_identical_with_demag(case, method):
    g, mat, omat, m0 = case
    kern = mx.DemagKernel.build(g, symmetric=True)
    rhs = mx.PartitionedRHS(mat, exchange=True, anisotropy=True, dmi=True, demag=kern, bias=(0, 0, 5e4))

    def run(env):
        st = mx.SimState(mx.VectorField3(g, m0.copy()))
        sim = mx.Simulation(st, rhs, mx.IntegratorSpec(method, 1e-14), sample_every=1, energy_in_samples=False)
        tr = with_env(env, lambda: sim.run_until(mx.StopCondition(max_steps=3)))
        return st.m.data.copy(), np.stack([tr.column(c) for c in ("mx", "my", "mz")], 1)

    m_t, tr_t = run({"MXB_ZTMA": "1"})
    m_s, tr_s = run({"MXB_ZTMA": "0"})
    assert np.array_equal(m_t, m_s)
    assert np.array_equal(tr_t, tr_s)
    # against the one-cell-per-thread kernels: same arithmetic per cell, the
    # per-step reductions are summed in another order
    m_c, tr_c = run({"MXB_ZMARCH": "0"})
    assert nrm(m_t, m_c) <= 1e-13
    assert np.max(np.abs(tr_t - tr_c)) <= 1e-12


def test_zmarch_edges_use_ghosts(case):
    """A tile column at the x edge: the TMA box starts two cells left of the
    grid (zero fill) and the ghost cells must replace every out-of-grid read."""
    g, mat, omat, _ = case
    m0 = np.zeros((3,) + g.shape)
    m0[2] = 8e5
    m0[0, :, :, 0] = 8e5 * 0.6
    m0[2, :, :, 0] = 8e5 * 0.8
    rhs = mx.PartitionedRHS(mat, exchange=True, dmi=True)
    terms = O.Terms(exchange=True, dmi=True)
    ref = O.h_eff(0.0, m0, omat, terms)
    for z in ("1", "0"):
        assert nrm(with_env({"MXB_ZTMA": z}, lambda: rhs.h_total_quiet(0.0, m0)), ref) <= 1e-12


@pytest.mark.parametrize("ztma", ["1", "0"])
def test_zmarch_ragged_tiles_match_oracle(ztma):
    """nx, ny, nz not multiples of the 32 x 8 x 16 tile: partial boxes at the
    far x edge (zero-filled past nx), partial y tiles and a short last z tile."""
    dims, cell = (200, 200, 70), (2e-9, 2.5e-9, 3e-9)
    g = mx.GridSpec(*dims, *cell)
    kw = dict(Ms=8e5, A=1.3e-11, Ku=4e5, eK=(0.3, -0.2, 1.0), D=2e-3, alpha=0.2)
    mat = mx.MaterialMap(g, **kw)
    omat = O.make_mat(dims, cell, **kw)
    m0 = O.renormalize(np.random.default_rng(11).normal(size=(3,) + g.shape), omat)
    bias = (2e4, 1e4, -3e4)
    rhs = mx.PartitionedRHS(mat, exchange=True, anisotropy=True, dmi=True, bias=bias)
    terms = O.Terms(exchange=True, anisotropy=True, dmi=True, bias=np.array(bias))
    plan = O.Plan(omat, terms.mode())
    f = lambda t, y: O.rhs_total(t, y, omat, terms, plan)
    env = {"MXB_ZTMA": ztma}
    assert nrm(with_env(env, lambda: rhs.h_total_quiet(0.0, m0)), O.h_eff(0.0, m0, omat, terms, plan)) <= 1e-12
    dt = 2e-14
    ref = O.renormalize(O.rk4_step(m0, 0.0, dt, f, lambda y: O.renormalize(y, omat)), omat)
    st = mx.SimState(mx.VectorField3(g, m0.copy()))
    sim = mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", dt), energy_in_samples=False)
    with_env(env, lambda: sim.run_until(mx.StopCondition(max_steps=1)))
    assert nrm(st.m.data, ref) <= 1e-12
