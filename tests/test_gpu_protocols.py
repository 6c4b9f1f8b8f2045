"""Reference protocols through the device loop (Simulation.run_until).

* a spatial, time-dependent bias (reference scenario.py:442-465 returns
  t -> (3,nz,ny,nx) for every spatial bias expression): the device loop
  uploads one field per stage evaluation (mxb_run_args.stage_bias_fields);
* muMAG SP4 field 1 on the reference's coarse grid (160x40x1, padded
  320x80, a radix-5 FFT length): the S-state preparation with the ramped
  diagonal field (a t -> (3,) callable, device stage-bias rows) at
  alpha = 0.5, then 2 ns of field 1 with energy samples every ~1 ps and the
  crossing time (reference bench/std4.py:67-200), against the reference's
  own run (tests/golden/make_golden.py sp4_protocol_golden).
"""
import numpy as np
import pytest

import paper_2602_12242_b200 as mx
from oracle import magnex_oracle as O
from tests.golden_io import load, spatial_case

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("method", ["rk4", "euler"])
def test_spatial_time_dependent_bias_matches_reference(method):
    z, omat, dt, bias = spatial_case(method)
    nx, ny, nz = omat.dims
    g = mx.GridSpec(nx, ny, nz, 2e-9, 2e-9, 2e-9)
    mat = mx.MaterialMap(g, Ms=z["Ms"], A=z["A"], Ku=z["Ku"], eK=z["eK"], alpha=z["alpha"])
    kern = mx.DemagKernel.from_packed(g, O.packed_tensor(nx, ny, nz, 2e-9, 2e-9, 2e-9))
    rhs = mx.PartitionedRHS(mat, exchange=True, anisotropy=True, demag=kern, bias=bias)
    st = mx.SimState(mx.VectorField3(g, z[method + "_m0"].copy()))
    tr = mx.Simulation(st, rhs, mx.IntegratorSpec(method, dt), sample_every=1,
                       energy_in_samples=True).run_until(mx.StopCondition(max_steps=20))
    got = np.stack([tr.column("mx"), tr.column("my"), tr.column("mz")], 1)
    assert np.max(np.abs(got - z[method + "_mean"])) <= 1e-12
    e = z[method + "_e_total"]
    assert np.max(np.abs(tr.column("e_total") - e)) <= 1e-10 * np.max(np.abs(e))
    assert np.max(np.abs(st.m.data - z[method + "_final"])) <= 1e-12 * 8e5
    # small stage-field chunks (several device calls per sample interval) give the same run
    st2 = mx.SimState(mx.VectorField3(g, z[method + "_m0"].copy()))
    sim = mx.Simulation(st2, rhs, mx.IntegratorSpec(method, dt), sample_every=7,
                        energy_in_samples=False)
    sim.STAGE_FIELD_BYTES = 1
    sim.run_until(mx.StopCondition(max_steps=20))
    assert np.array_equal(st2.m.data, st.m.data)


def ramped_bias(vec, hold, ramp):
    """bench/std4.py:67-79"""
    v = np.asarray(vec, dtype=np.float64)

    def bias(t):
        if t <= hold:
            return v
        if t < hold + ramp:
            return v * (1.0 - (t - hold) / ramp)
        return np.zeros(3)
    return bias


def crossing_time(t, mx_):
    """bench/std4.py:191-200"""
    s = np.sign(mx_)
    for i in range(len(mx_) - 1):
        if s[i] > 0 and s[i + 1] <= 0:
            if mx_[i] == mx_[i + 1]:
                return float(t[i + 1])
            f = mx_[i] / (mx_[i] - mx_[i + 1])
            return float(t[i] + f * (t[i + 1] - t[i]))
    return None


def sp4_protocol(kernel_of):
    """std4.prepare_s_state + run_std4(1, 'coarse') through this package."""
    d = 3.125e-9
    g = mx.GridSpec(160, 40, 1, d, d, d)
    dt = O.stable_dt(d, 1.3e-11, 8e5, 0.5)
    kern = kernel_of(g)
    # S-state: alpha 0.5, +x, (1e5,1e5,1e5) for 20 ps ramped off over 10 ps, relax up to 1 ns
    mat = mx.MaterialMap(g, Ms=8e5, A=1.3e-11, alpha=0.5)
    rhs = mx.PartitionedRHS(mat, exchange=True, demag=kern,
                            bias=ramped_bias((1e5, 1e5, 1e5), 20e-12, 10e-12))
    m = np.zeros((3,) + g.shape)
    m[0] = 8e5
    st = mx.SimState(mx.VectorField3(g, m))
    sim = mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", dt), sample_every=10_000_000,
                        energy_in_samples=False)
    sim.run_until(mx.StopCondition(max_time=30e-12))
    sim.run_until(mx.StopCondition(max_time=30e-12 + 1e-9, equilibrium_tol=1e-9))
    s_state = st.m.data.copy()
    # field 1 at alpha 0.02, samples every ~1 ps with energies and a sample callback
    mat = mx.MaterialMap(g, Ms=8e5, A=1.3e-11, alpha=0.02)
    rhs = mx.PartitionedRHS(mat, exchange=True, demag=kern, bias=np.array([-19576.0, 3422.0, 0.0]))
    st = mx.SimState(mx.VectorField3(g, s_state.copy()))
    snap = {}

    def on_sample(s, row):
        if row["mx"] < 0.0 and "m" not in snap:
            snap["t"] = s.t

    sim = mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", dt), sample_every=max(1, round(1e-12 / dt)),
                        sample_callback=on_sample, energy_in_samples=True)
    tr = sim.run_until(mx.StopCondition(max_time=2e-9))
    return s_state, tr, snap


def test_sp4_full_protocol_matches_reference():
    z = load("sp4_protocol")
    packed = O.packed_tensor(160, 40, 1, 3.125e-9, 3.125e-9, 3.125e-9)
    s_state, tr, snap = sp4_protocol(lambda g: mx.DemagKernel.from_packed(g, packed))
    e_s = float(np.max(np.abs(s_state - z["s_state"])) / 8e5)
    dm = max(float(np.max(np.abs(tr.column(k) - z[k]))) for k in ("mx", "my", "mz"))
    tc = crossing_time(tr.column("t"), tr.column("mx"))
    print(f"SP4 protocol (reference tensor): S-state {e_s:.3e}, <m>(t) {dm:.3e}, "
          f"crossing {tc!r} vs {float(z['crossing_time'])!r}")
    assert len(tr.samples) == len(z["t"])
    assert np.array_equal(tr.column("t"), z["t"])
    assert np.array_equal(tr.column("n_demag_evals"), z["n_demag"])
    assert e_s <= 1e-9
    assert dm <= 1e-6          # north-star contract (observed value printed)
    assert abs(tc - float(z["crossing_time"])) <= 1e-15
    assert np.max(np.abs(tr.column("e_total") - z["e_total"])) <= 1e-6 * np.max(np.abs(z["e_total"]))
    assert snap["t"] >= tc


def test_sp4_full_protocol_gpu_built_tensor():
    """The same protocol with the tensor built on the GPU (DemagKernel.build):
    the tensor differs from the reference's at its libm noise floor
    (tests/test_tensor_noise_floor.py); <m>(t) is held to the contract."""
    z = load("sp4_protocol")
    s_state, tr, _ = sp4_protocol(lambda g: mx.DemagKernel.build(g))
    dm = max(float(np.max(np.abs(tr.column(k) - z[k]))) for k in ("mx", "my", "mz"))
    tc = crossing_time(tr.column("t"), tr.column("mx"))
    print(f"SP4 protocol (GPU tensor): <m>(t) {dm:.3e}, crossing {tc!r} vs {float(z['crossing_time'])!r}")
    assert dm <= 1e-6
    assert abs(tc - float(z["crossing_time"])) <= 1e-15 + 1e-6 * float(z["crossing_time"])
