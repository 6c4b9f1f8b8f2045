"""Behavioural checks of the B200 package, modelled on the reference's own test
strategy (pkg/tests: closed forms, contracts and properties) and
run against paper_2602_12242_b200 on the GPU."""
import math

import numpy as np
import pytest

import paper_2602_12242_b200 as mx
from oracle import magnex_oracle as O

pytestmark = pytest.mark.gpu
MS = 8e5
rng = np.random.default_rng(2024)


# ---------------------------------------------------------------- fields ----
def test_uniaxial_field_along_easy_axis():
    g = mx.GridSpec(3, 2, 1, 3e-9, 3e-9, 3e-9)
    ku = 0.1 * 0.5 * mx.MU0 * MS ** 2
    mat = mx.MaterialMap(g, Ms=MS, Ku=ku, eK=(0, 0, 1))
    h = mx.anisotropy_field(mx.VectorField3.from_uniform(g, (0, 0, MS)), mat)
    assert np.allclose(h[2], 2 * ku / (mx.MU0 * MS), rtol=1e-13)
    assert np.all(h[:2] == 0.0)
    assert np.all(mx.anisotropy_field(mx.VectorField3.from_uniform(g, (MS, 0, 0)), mat) == 0.0)


def test_exchange_pair_and_uniform_state():
    g = mx.GridSpec(2, 1, 1, 3e-9, 3e-9, 3e-9)
    A = 1.3e-11
    mat = mx.MaterialMap(g, Ms=MS, A=A)
    m = mx.VectorField3.zeros(g)
    m.data[:, 0, 0, 0] = (MS, 0, 0)
    m.data[:, 0, 0, 1] = (0, MS, 0)
    h = mx.exchange_field(m, mat)
    pref = 2 * A / (mx.MU0 * MS ** 2) / g.dx ** 2
    assert np.allclose(h[:, 0, 0, 0], pref * (m.data[:, 0, 0, 1] - m.data[:, 0, 0, 0]), rtol=1e-12)
    g3 = mx.GridSpec(5, 4, 3, 2e-9, 3e-9, 4e-9)
    mat3 = mx.MaterialMap(g3, Ms=MS, A=A)
    assert np.allclose(mx.exchange_field(mx.VectorField3.from_uniform(g3, (3e5, -4e5, 1e5)), mat3), 0,
                       atol=1e-20)


def test_exchange_helix_is_an_eigenvector_in_periodic_mode():
    nx, dx, A = 16, 2e-9, 1.005154e-11
    g = mx.GridSpec(nx, 1, 1, dx, dx, dx)
    mat = mx.MaterialMap(g, Ms=MS, A=A)
    k = 2 * np.pi * 3 / (nx * dx)
    x = (np.arange(nx) + 0.5) * dx
    m = mx.VectorField3.zeros(g)
    m.data[0, 0, 0] = MS * np.cos(k * x)
    m.data[1, 0, 0] = MS * np.sin(k * x)
    lam = -(2 * A / (mx.MU0 * MS ** 2)) * (2 - 2 * np.cos(k * dx)) / dx ** 2
    assert np.allclose(mx.exchange_field(m, mat, ghost_mode="periodic"), lam * m.data, rtol=1e-10,
                       atol=1e-6)


def test_exchange_linear_and_self_adjoint():
    g = mx.GridSpec(6, 5, 4, 2e-9, 2.5e-9, 3e-9)
    mat = mx.MaterialMap(g, Ms=MS, A=1.3e-11)
    u, v = rng.normal(size=(2, 3) + g.shape)
    Lu = mx.exchange_field(mx.VectorField3(g, u), mat, ghost_mode="periodic")
    Lv = mx.exchange_field(mx.VectorField3(g, v), mat, ghost_mode="periodic")
    assert np.dot(u.ravel(), Lv.ravel()) == pytest.approx(np.dot(Lu.ravel(), v.ravel()), rel=1e-10)
    Luv = mx.exchange_field(mx.VectorField3(g, 2 * u - 0.5 * v), mat, ghost_mode="periodic")
    assert np.allclose(Luv, 2 * Lu - 0.5 * Lv, rtol=1e-12, atol=1e-9)


def test_vacuum_gap_isolates_cells():
    g = mx.GridSpec(3, 1, 1, 2e-9, 2e-9, 2e-9)
    mat = mx.MaterialMap(g, Ms=np.array([[[MS, 0.0, MS]]]), A=1.3e-11)
    m = mx.VectorField3.zeros(g)
    m.data[0, 0, 0, 0] = MS
    m.data[1, 0, 0, 2] = MS
    assert np.allclose(mx.exchange_field(m, mat), 0.0)


def test_dmi_zero_d_is_zero_and_matches_neumann_exchange():
    g = mx.GridSpec(4, 4, 1, 1e-9, 1e-9, 1e-9)
    mat = mx.MaterialMap(g, Ms=1.1e6, A=16e-12, D=0.0)
    m = mx.VectorField3(g, rng.normal(size=(3,) + g.shape) * 1.1e6)
    assert np.all(mx.dmi_field(m, mat) == 0.0)
    assert np.allclose(mx.exchange_field(m, mat, "dmi"), mx.exchange_field(m, mat, "neumann"))


def test_energies_closed_forms():
    g = mx.GridSpec(3, 3, 2, 2e-9, 2e-9, 2e-9)
    ku, A = 4.021216e4, 1.005154e-11
    mat = mx.MaterialMap(g, Ms=MS, A=A, Ku=ku, eK=(0, 0, 1))
    e = mx.energy_breakdown(mx.VectorField3.from_uniform(g, (0, 0, MS)), mat)
    assert e.e_exch == 0.0 and abs(e.e_anis) < 1e-20
    m = mx.VectorField3.from_uniform(g, (MS, 0, 0))
    assert mx.energy_breakdown(m, mat).e_anis == pytest.approx(ku, rel=1e-12)
    e = mx.energy_breakdown(m, mat, h_bias=np.array([1e5, 0, 0]))
    assert e.e_zeeman == pytest.approx(-mx.MU0 * MS * 1e5, rel=1e-12)
    nx, dx = 32, 2e-9
    g1 = mx.GridSpec(nx, 1, 1, dx, dx, dx)
    mat1 = mx.MaterialMap(g1, Ms=MS, A=A)
    k = 2 * np.pi / (nx * dx)
    x = (np.arange(nx) + 0.5) * dx
    h = mx.VectorField3.zeros(g1)
    h.data[0, 0, 0], h.data[1, 0, 0] = MS * np.cos(k * x), MS * np.sin(k * x)
    e = mx.energy_breakdown(h, mat1, ghost_mode="periodic")
    assert e.e_exch == pytest.approx(A * (np.sin(k * dx) / dx) ** 2, rel=1e-10)


# ----------------------------------------------------------------- demag ----
@pytest.mark.parametrize("dims,cell", [((1, 1, 1), (1e-9,) * 3), ((2, 2, 2), (1e-9,) * 3),
                                       ((6, 5, 4), (1e-9, 2e-9, 1.5e-9)), ((8, 1, 1), (2e-9, 1e-9, 3e-9)),
                                       ((6, 5, 1), (1.5e-9,) * 3), ((8, 8, 8), (1e-9,) * 3)])
def test_gpu_built_fft_matches_direct_sum(dims, cell):
    g = mx.GridSpec(*dims, *cell)
    m = rng.normal(size=(3,) + g.shape) * 8e5
    h = mx.DemagKernel.build(g).field(m)
    ref = O.demag_direct(m, O.tensor_elements(*dims, *cell))
    assert np.max(np.abs(h - ref)) <= 1e-9 * np.max(np.abs(ref))


def test_uniform_cube_centre_field_is_minus_third():
    g = mx.GridSpec(9, 9, 9, 2e-9, 2e-9, 2e-9)
    mat = mx.MaterialMap(g, Ms=MS)
    m = mx.VectorField3.from_uniform(g, (0, 0, MS))
    h = mx.demag_field_fft(m, mx.DemagKernel.build(g))
    assert h[2, 4, 4, 4] == pytest.approx(-MS / 3, rel=0.01)
    assert abs(h[0, 4, 4, 4]) < 1e-9 * MS and abs(h[1, 4, 4, 4]) < 1e-9 * MS
    e = mx.energy_breakdown(m, mat, h_demag=h)
    assert e.e_demag == pytest.approx(0.5 * mx.MU0 * MS ** 2 / 3, rel=0.02)


def test_demag_energy_is_non_negative_and_deterministic():
    g = mx.GridSpec(5, 4, 3, 1e-9, 1e-9, 2e-9)
    mat = mx.MaterialMap(g, Ms=MS)
    k = mx.DemagKernel.build(g)
    for _ in range(4):
        m = mx.VectorField3(g, rng.normal(size=(3,) + g.shape) * MS)
        h = k.field(m.data)
        assert np.array_equal(h, k.field(m.data))
        assert mx.energy_breakdown(m, mat, h_demag=h).e_demag >= 0.0
    assert np.array_equal(k.spectra, mx.DemagKernel.build(g).spectra)
    with pytest.raises(ValueError, match="kernel built for"):
        mx.demag_field_fft(mx.VectorField3.zeros(mx.GridSpec(3, 3, 3, 1e-9, 1e-9, 1e-9)), k)


def test_vacuum_sources_are_transparent_and_origin_is_irrelevant():
    g = mx.GridSpec(6, 4, 2, 1e-9, 1e-9, 1e-9)
    m = np.zeros((3,) + g.shape)
    m[:, :, :, :3] = rng.normal(size=(3, 2, 4, 3)) * MS
    h_full = mx.DemagKernel.build(g).field(m)
    gs = mx.GridSpec(3, 4, 2, 1e-9, 1e-9, 1e-9)
    h_sub = mx.DemagKernel.build(gs).field(np.ascontiguousarray(m[:, :, :, :3]))
    assert np.allclose(h_full[:, :, :, :3], h_sub, rtol=1e-12, atol=1e-6)
    g1 = mx.GridSpec(4, 4, 1, 2e-9, 2e-9, 2e-9)
    g2 = mx.GridSpec(4, 4, 1, 2e-9, 2e-9, 2e-9, origin=(5e-8, -3e-8, 1e-9))
    d = rng.normal(size=(3,) + g1.shape) * MS
    assert np.array_equal(mx.DemagKernel.build(g1).field(d), mx.DemagKernel.build(g2).field(d))


def test_dipole_switch_continuity_of_gpu_tensor():
    n = 120
    xx = mx.tensor_elements(n, 1, 1, 1e-9, 1e-9, 1e-9)[0, 0, 0]
    for disp in (58, 59, 61, 63):
        dip = 2.0 / (4 * np.pi * disp ** 3)
        assert abs(xx[n - 1 + disp] - dip) / dip < 1e-3


# ------------------------------------------------------------------- llg ----
def single_spin(alpha, m0=(MS, 0.0, 0.0), h0=7.9577e5):
    g = mx.GridSpec(1, 1, 1, 1e-9, 1e-9, 1e-9)
    mat = mx.MaterialMap(g, Ms=MS, alpha=alpha)
    rhs = mx.PartitionedRHS(mat, exchange=False, bias=(0.0, 0.0, h0))
    return g, mat, rhs, mx.SimState(mx.VectorField3.from_uniform(g, m0)), h0


def closed_form(t, alpha, h0):
    gl = 1.759e11 / (1 + alpha * alpha)
    om = gl * mx.MU0 * h0
    th = 2 * math.atan(math.exp(-alpha * om * t))
    return MS * np.array([math.sin(th) * math.cos(om * t), math.sin(th) * math.sin(om * t),
                          math.cos(th)])


def test_torque_signs_and_toggles():
    g, mat, rhs, st, _ = single_spin(0.5, m0=(0, 0, MS))
    assert np.all(rhs.rhs_total(0.0, st.m.data) == 0.0)
    _, _, rhs, st, _ = single_spin(0.02)
    out = rhs.rhs_total(0.0, st.m.data)[:, 0, 0, 0]
    assert out[1] > 0 and out[2] > 0
    rhs.precession = False          # toggled after construction, like the reference tests
    out = rhs.rhs_total(0.0, st.m.data)[:, 0, 0, 0]
    assert out[1] == 0.0 and out[2] > 0
    rhs.precession, rhs.damping = True, False
    out = rhs.rhs_total(0.0, st.m.data)[:, 0, 0, 0]
    assert out[1] > 0 and out[2] == 0.0
    _, _, rhs0, st0, _ = single_spin(0.0)
    o0 = rhs0.rhs_total(0.0, st0.m.data)
    assert abs(float(np.sum(o0 * st0.m.data))) < 1e-20


def test_vacuum_torque_is_zero():
    g = mx.GridSpec(3, 1, 1, 1e-9, 1e-9, 1e-9)
    mat = mx.MaterialMap(g, Ms=np.array([[[MS, 0.0, MS]]]), alpha=0.1)
    m = mx.VectorField3.zeros(g)
    m.data[0, :, :, 0] = MS
    m.data[2, :, :, 2] = MS
    out = mx.llg_rhs(m, mx.VectorField3.from_uniform(g, (0.0, 1e5, 0.0)), mat)
    assert np.all(out.data[:, 0, 0, 1] == 0.0) and np.any(out.data[:, 0, 0, 0] != 0.0)


@pytest.mark.parametrize("alpha,dt,t_end,tol", [(0.0, 1e-13, 1e-11, 1e-7), (0.5, 5e-14, 2e-11, 1e-6)])
def test_single_spin_closed_form(alpha, dt, t_end, tol):
    g, mat, rhs, st, h0 = single_spin(alpha)
    mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", dt, renorm_each_stage=False),
                  sample_every=10 ** 9, energy_in_samples=False).run_until(mx.StopCondition(max_time=t_end))
    assert np.max(np.abs(st.m.data[:, 0, 0, 0] - closed_form(t_end, alpha, h0))) < tol * MS


def test_rk4_is_fourth_order():
    errs = []
    for dt in (4e-13, 2e-13, 1e-13):
        g, mat, rhs, st, h0 = single_spin(0.2)
        mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", dt, renorm_each_stage=False),
                      sample_every=10 ** 9, energy_in_samples=False).run_until(
            mx.StopCondition(max_time=4e-12))
        errs.append(np.max(np.abs(st.m.data[:, 0, 0, 0] - closed_form(4e-12, 0.2, h0))) / MS)
    assert abs(math.log2(errs[1] / errs[2]) - 4.0) < 0.15, errs


def film(alpha=0.1):
    g = mx.GridSpec(4, 4, 1, 2e-9, 2e-9, 2e-9)
    mat = mx.MaterialMap(g, Ms=MS, alpha=alpha, A=1.3e-11)
    rhs = mx.PartitionedRHS(mat, exchange=True, demag=mx.DemagKernel.build(g), bias=(0.0, 0.0, 1e4))
    m = mx.VectorField3(g, np.random.default_rng(7).normal(size=(3,) + g.shape))
    mx.renormalize(m, mat)
    return g, mat, rhs, mx.SimState(m)


def test_counter_contracts_and_accumulation():
    g, mat, rhs, st = film()
    tr = mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", 2.5e-14), sample_every=10 ** 9,
                       energy_in_samples=False).run_until(mx.StopCondition(max_time=1.25e-13))
    assert st.step == 5 and tr.stop_reason == "max_time"
    assert tr.counters == {"exchange": 20, "demag": 20, "bias": 20}
    g, mat, rhs, st = film()
    sim = mx.Simulation(st, rhs, mx.IntegratorSpec("euler", 1e-15), sample_every=10 ** 9,
                        energy_in_samples=False)
    sim.run_until(mx.StopCondition(max_steps=7))
    assert rhs.counters["demag"] == 7
    sim.run_until(mx.StopCondition(max_steps=5))
    assert rhs.counters["demag"] == 12


def test_norm_is_ms_within_four_ulp_after_steps():
    g, mat, rhs, st = film(alpha=0.5)
    mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", 1e-13), sample_every=10 ** 9,
                  energy_in_samples=False).run_until(mx.StopCondition(max_steps=20))
    assert np.max(np.abs(st.m.norm() - MS)) <= 4 * np.spacing(MS)


def test_stop_reasons():
    g, mat, rhs, st, _ = single_spin(0.5, m0=(0, 0, MS))
    tr = mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", 1e-13), energy_in_samples=False).run_until(
        mx.StopCondition(max_steps=100, equilibrium_tol=1e-9))
    assert tr.stop_reason == "equilibrated" and st.step == 1
    g, mat, rhs, st, _ = single_spin(0.0)
    tr = mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", 1e-13), energy_in_samples=False).run_until(
        mx.StopCondition(max_steps=5, equilibrium_tol=1e-9))
    assert tr.stop_reason == "not_converged" and st.step == 5


def test_energy_decreases_during_damped_relaxation():
    g, mat, rhs, st = film(alpha=0.8)
    tr = mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", 2e-13), sample_every=1).run_until(
        mx.StopCondition(max_steps=40))
    e = tr.column("e_total")
    assert np.all(np.diff(e) / np.maximum(np.abs(e[:-1]), 1e-30) <= 1e-6) and e[-1] < e[0]


def test_blowup_is_detected():
    g = mx.GridSpec(2, 1, 1, 1e-9, 1e-9, 1e-9)
    mat = mx.MaterialMap(g, Ms=MS, alpha=0.5, A=1.3e-11)
    m = mx.VectorField3.zeros(g)
    m.data[0, 0, 0, 0] = MS
    m.data[1, 0, 0, 1] = MS
    sim = mx.Simulation(mx.SimState(m), mx.PartitionedRHS(mat), mx.IntegratorSpec("euler", 1e-12),
                        energy_in_samples=False)
    with pytest.raises(mx.IntegrationBlowup):
        sim.run_until(mx.StopCondition(max_steps=50))


def test_bias_sampled_at_stage_times():
    seen = []

    def ramp(t):
        seen.append(t)
        return np.array([0.0, 0.0, 1e5 * t / 1e-12])

    g = mx.GridSpec(1, 1, 1, 1e-9, 1e-9, 1e-9)
    mat = mx.MaterialMap(g, Ms=MS, alpha=0.3)
    rhs = mx.PartitionedRHS(mat, exchange=False, bias=ramp)
    st = mx.SimState(mx.VectorField3.from_uniform(g, (MS, 0.0, 0.0)))
    mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", 1e-13), sample_every=10 ** 9,
                  energy_in_samples=False).run_until(mx.StopCondition(max_steps=1))
    assert seen[:4] == [0.0, 5e-14, 5e-14, 1e-13]


def test_sampling_cadence_and_csv(tmp_path):
    g, mat, rhs, st = film(alpha=0.5)
    tr = mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", 1e-13), sample_every=3).run_until(
        mx.StopCondition(max_steps=10))
    assert np.allclose(tr.column("t"), [0.0, 3e-13, 6e-13, 9e-13, 1e-12])
    from paper_2602_12242_b200.io import CSV_COLUMNS, read_timeseries_csv
    p = tmp_path / "traj.csv"
    tr.write_csv(p)
    cols = read_timeseries_csv(p)
    assert list(cols) == CSV_COLUMNS and cols["n_demag_evals"][-1] == 40


def test_quiet_diagnostics_leave_counters():
    g, mat, rhs, st = film()
    before = dict(rhs.counters)
    rhs.h_total_quiet(0.0, st.m.data)
    rhs.demag_quiet(st.m.data)
    rhs.energies(0.0, st.m)
    assert rhs.counters == before


def test_precession_off_reaches_the_same_fixed_point():
    def relax(prec):
        g = mx.GridSpec(2, 2, 1, 2e-9, 2e-9, 2e-9)
        mat = mx.MaterialMap(g, Ms=MS, alpha=0.9, A=1.3e-11)
        rhs = mx.PartitionedRHS(mat, exchange=True, demag=mx.DemagKernel.build(g),
                                bias=(6e4, 2e4, 3e4), precession=prec)
        m = mx.VectorField3(g, np.random.default_rng(7).normal(size=(3,) + g.shape))
        mx.renormalize(m, mat)
        st = mx.SimState(m)
        tr = mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", 5e-13), sample_every=10 ** 9,
                           energy_in_samples=False).run_until(
            mx.StopCondition(max_steps=30000, equilibrium_tol=1e-9))
        assert tr.stop_reason == "equilibrated"
        return mx.mean_normalized(st.m, mat)

    assert np.max(np.abs(relax(True) - relax(False))) < 1e-4


# ------------------------------------------------------------------ grid ----
def test_renormalize_contracts():
    g = mx.GridSpec(5, 4, 3, 2e-9, 2e-9, 2e-9)
    mat = mx.MaterialMap(g, Ms=MS)
    m = mx.VectorField3(g, rng.normal(size=(3,) + g.shape))
    mx.renormalize(m, mat)
    assert np.all(np.abs(m.norm() - MS) <= 4 * np.spacing(MS))
    before = m.data.copy()
    mx.renormalize(m, mat)
    assert np.all(np.abs(m.data - before) <= np.spacing(np.abs(before)))
    g3 = mx.GridSpec(3, 1, 1, 2e-9, 2e-9, 2e-9)
    mat3 = mx.MaterialMap(g3, Ms=np.array([[[MS, 0.0, MS]]]))
    m3 = mx.VectorField3.from_uniform(g3, (1e5, 2e5, 0.0))
    mx.renormalize(m3, mat3)
    assert np.all(m3.data[:, 0, 0, 1] == 0.0)
    m3.data[:, 0, 0, 2] = 0.0
    with pytest.raises(mx.RenormalizeError, match=r"i=2"):
        mx.renormalize(m3, mat3)


def test_mean_excludes_vacuum():
    g = mx.GridSpec(4, 1, 1, 2e-9, 2e-9, 2e-9)
    mat = mx.MaterialMap(g, Ms=np.array([[[MS, MS, 0.0, MS]]]))
    m = mx.VectorField3.zeros(g)
    m.data[0, 0, 0, 0], m.data[0, 0, 0, 1], m.data[2, 0, 0, 3] = MS, -MS, MS
    assert mx.mean_normalized(m, mat) == pytest.approx([0.0, 0.0, 1.0 / 3.0])
    with pytest.raises(ValueError):
        mx.mean_normalized(m, mx.MaterialMap(g, Ms=0.0))
