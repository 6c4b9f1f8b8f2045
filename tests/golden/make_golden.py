"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports ``magnex`` read-only from /root/reference/pkg/src and writes
``tests/golden/*.npz``.  The fixtures pin the CPU oracle (oracle/magnex_oracle.py)
and, through it, the CUDA path.  Versions used are recorded in each file
(``numpy``/``scipy`` keys).  Large arrays that the oracle regenerates exactly
(packed demag tensors) are pinned by sha256 instead of being stored.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np
import scipy

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from magnex import demag as rdemag  # noqa: E402
from magnex.grid import GridSpec, MaterialMap, VectorField3, mean_normalized, renormalize  # noqa: E402
from magnex.fields import energy_breakdown  # noqa: E402
from magnex.integrators import euler_step, rk4_step  # noqa: E402
from magnex.llg import (IntegratorSpec, PartitionedRHS, SimState, Simulation,  # noqa: E402
                        StopCondition)

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def case(name, dims, cell, mat_kw, terms, seed, *, ghost_mode=None, bias=None,
         demag=False, dt=1e-13, nsteps=0, method="rk4", msmap=None, store_tensor=True,
         mri_steps=0):
    nx, ny, nz = dims
    g = GridSpec(nx, ny, nz, *cell)
    kw = dict(mat_kw)
    if msmap is not None:
        kw["Ms"] = msmap(g)
    mat = MaterialMap(g, **kw)
    rng = np.random.default_rng(seed)
    m = VectorField3(g, rng.normal(size=(3,) + g.shape))
    renormalize(m, mat)
    m0 = m.data.copy()
    kern = rdemag.DemagKernel.build(g) if demag else None
    rhs = PartitionedRHS(mat, exchange="exchange" in terms, anisotropy="anisotropy" in terms,
                         dmi="dmi" in terms, demag=kern, bias=bias, ghost_mode=ghost_mode)
    out = {"dims": np.array(dims), "cell": np.array(cell), "m0": m0, "dt": dt,
           "Ms": mat.Ms, "A": mat.A, "Ku": mat.Ku, "D": mat.D, "alpha": mat.alpha,
           "eK": mat.eK, "terms": np.array(sorted(terms)),
           "ghost_mode": rhs.ghost_mode,
           "bias": np.zeros(3) if bias is None else np.asarray(bias, dtype=np.float64),
           "has_bias": bias is not None, "has_demag": demag,
           "numpy": np.__version__, "scipy": scipy.__version__}
    for t, op in rhs._ops.items():
        out["h_" + t] = op(m0)
    out["h_total"] = rhs.h_total_quiet(0.0, m0)
    out["rhs_total"] = rhs.rhs_total(0.0, m0)
    if demag:
        if store_tensor:
            out["packed"] = kern._packed
        out["packed_sha"] = sha(kern._packed)
        out["spectra_sha"] = sha(kern.spectra)

    def hook(y):
        f = VectorField3(g, y)
        renormalize(f, mat)
        return f.data

    out["rk4_step"] = rk4_step(m0, 0.0, dt, rhs.rhs_total, hook)
    out["euler_step"] = euler_step(m0, 0.0, dt, rhs.rhs_total)
    e = energy_breakdown(VectorField3(g, m0), mat, h_demag=rhs.demag_quiet(m0),
                         h_bias=rhs.bias_at(0.0), plan=rhs.plan)
    out["energies"] = np.array([e.e_demag, e.e_exch, e.e_anis, e.e_zeeman])
    if nsteps:
        st = SimState(VectorField3(g, m0.copy()))
        sim = Simulation(st, rhs, IntegratorSpec(method, dt), sample_every=1,
                         energy_in_samples=False)
        tr = sim.run_until(StopCondition(max_steps=nsteps))
        out["trace_t"] = tr.column("t")
        out["trace_m"] = np.stack([tr.column("mx"), tr.column("my"), tr.column("mz")], 1)
        out["trace_final"] = st.m.data.copy() if g.n_cells <= 20000 else np.zeros(0)
        out["trace_final_sha"] = sha(st.m.data)
        out["trace_method"] = method
        if bool(mri_steps) and "exchange" in terms:
            rhs.counters = {k: 0 for k in rhs.counters}
            st = SimState(VectorField3(g, m0.copy()))
            sim = Simulation(st, rhs, IntegratorSpec("mri-kw3", 4 * dt), sample_every=1,
                             energy_in_samples=False)
            tr = sim.run_until(StopCondition(max_steps=mri_steps))
            out["mri_dt"] = 4 * dt
            out["mri_trace_m"] = np.stack([tr.column("mx"), tr.column("my"), tr.column("mz")], 1)
            out["mri_final"] = st.m.data.copy()
            out["mri_counters"] = np.array([tr.counters.get(k, 0) for k in
                                            ("exchange", "anisotropy", "dmi", "demag", "bias")])
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **out)
    print(name, "ok", {k: (v.shape if hasattr(v, "shape") else v) for k, v in out.items()
                       if k.startswith(("h_", "rk4", "trace_m"))})


def disk(g):
    X, Y, _ = g.cell_centers()
    cx = 0.5 * g.nx * g.dx
    R = 0.5 * g.nx * g.dx
    return np.where((X - cx) ** 2 + (Y - cx) ** 2 <= R * R, 1.1e6, 0.0)


SPATIAL_SCENARIO = """\
[grid]
nx = 12
ny = 10
nz = 2
dx = 2e-9
dy = 2e-9
dz = 2e-9
[material]
ms = 8e5
aex = 1.3e-11
alpha = 0.1
ku = 3e4
[physics]
exchange = true
demag = true
anisotropy = true
[bias]
hx = "2e4 * sin(2 * pi * x / 24e-9) * cos(2 * pi * t / 5e-13)"
hy = "where(y > 10e-9, 5e3, -5e3)"
hz = "1e4 * exp(-t / 2e-13) + 1e3 * z / 4e-9"
[initial]
mx = "cos(x / 6e-9)"
my = "sin(x / 6e-9)"
mz = "0.2"
[integrator]
method = rk4
dt = 1e-14
[stop]
max_steps = 20
[output]
sample_every = 1
energies = true
"""


def spatial_bias_golden():
    """A scenario whose bias is a spatial, time-dependent expression: the
    reference's ScenarioConfig.build_bias returns t -> (3,nz,ny,nx)
    (scenario.py:442-465).  The bias field of every stage evaluation is
    recorded (so the test can replay it bit for bit) with the run's trace."""
    from magnex.scenario import loads
    out = {}
    for method, dt in (("rk4", 1e-14), ("euler", 5e-15)):
        cfg = loads(SPATIAL_SCENARIO.replace("method = rk4", f"method = {method}")
                    .replace("dt = 1e-14", f"dt = {dt!r}"))
        sim = cfg.build_simulation()
        bias = sim.rhs._bias
        assert callable(bias)
        seen = {}

        def rec(t, _b=bias, _seen=seen):
            v = _b(t)
            _seen.setdefault(float(t), v.copy())
            return v

        sim.rhs._bias = rec
        m0 = sim.state.m.data.copy()
        tr = sim.run_until(cfg.stop)
        ts = np.array(sorted(seen))
        out[method + "_m0"] = m0
        out[method + "_times"] = ts
        out[method + "_fields"] = np.stack([seen[t] for t in ts])
        out[method + "_mean"] = np.stack([tr.column("mx"), tr.column("my"), tr.column("mz")], 1)
        out[method + "_e_total"] = tr.column("e_total")
        out[method + "_final"] = sim.state.m.data.copy()
        out[method + "_dt"] = dt
    mat = loads(SPATIAL_SCENARIO).build_material()
    out["Ms"], out["A"], out["Ku"], out["alpha"], out["eK"] = mat.Ms, mat.A, mat.Ku, mat.alpha, mat.eK
    out["scenario"] = np.array(SPATIAL_SCENARIO)
    np.savez_compressed(os.path.join(OUT, "spatial_bias.npz"), **out)
    print("spatial_bias ok", out["rk4_fields"].shape)


def sp4_protocol_golden():
    """muMAG SP4 field 1 on the reference's coarse grid (160x40x1, 3.125 nm,
    padded 320x80: radix 5) through the reference's own driver: S-state
    preparation with ramped_bias at alpha = 0.5 (30 ps + relaxation up to
    1 ns at the equilibrium tolerance), then 2 ns of field 1 at alpha = 0.02
    with energy samples every ~1 ps (bench/std4.py:67-188) and crossing_time
    (bench/std4.py:191-200)."""
    from magnex.bench import std4
    p = std4.Std4Params()
    s_state = std4.prepare_s_state("coarse", p, emit=print)
    res, checks = std4.run_std4(1, "coarse", p, s_state=s_state, emit=print)
    tr = res.trajectory
    np.savez_compressed(os.path.join(OUT, "sp4_protocol.npz"),
                        s_state=s_state.data, t=tr.column("t"), mx=tr.column("mx"),
                        my=tr.column("my"), mz=tr.column("mz"), e_total=tr.column("e_total"),
                        e_demag=tr.column("e_demag"), e_exch=tr.column("e_exch"),
                        n_demag=tr.column("n_demag_evals"),
                        crossing_time=np.nan if res.crossing_time is None else res.crossing_time,
                        stop_reason=np.array(tr.stop_reason),
                        numpy=np.__version__, scipy=scipy.__version__)
    print("sp4_protocol ok, crossing", res.crossing_time, "samples", len(tr.samples))


def radix5_goldens():
    """Padded lengths with a factor 5 (2n padding, demag.py:152-155): the
    100x100 DMI disk with demag (skyrmion benchmark, 200x200) and the SP4
    coarse grid (160x40x1 -> 320x80)."""
    ALL = ("exchange", "anisotropy", "dmi")
    case("dmi_disk_100_demag", (100, 100, 1), (1e-9, 1e-9, 0.25e-9),
         dict(A=16e-12, Ku=5.5e5, D=4.5e-3, alpha=1.0), ALL, 16, msmap=disk, demag=True,
         dt=1e-14, nsteps=10, store_tensor=False)
    d = 3.125e-9
    case("sp4_160x40x1", (160, 40, 1), (d, d, 3e-9),
         dict(Ms=8e5, A=1.3e-11, alpha=0.02), ("exchange",), 17,
         bias=(-19576.0, 3422.0, 0.0), demag=True, dt=2e-13, nsteps=20, store_tensor=False)


def bench32_golden():
    """The bench's material and cell (bench.py setup_problem) at 32^3 with a
    random-direction m: the reference's H_demag (its own tensor) and H_eff.
    bench.py reports its GPU-built tensor's deviation from these at run time."""
    g = GridSpec(32, 32, 32, 4e-9, 4e-9, 4e-9)
    mat = MaterialMap(g, Ms=8e5, A=1.3e-11, Ku=5e4, eK=(0.0, 0.0, 1.0), D=1e-3, alpha=0.1)
    rng = np.random.default_rng(25)
    m = rng.standard_normal((3,) + g.shape)
    m *= 8e5 / np.sqrt((m * m).sum(axis=0))
    kern = rdemag.DemagKernel.build(g)
    rhs = PartitionedRHS(mat, exchange=True, anisotropy=True, dmi=True, demag=kern,
                         bias=np.array([1e4, 0.0, 0.0]))
    np.savez_compressed(os.path.join(OUT, "bench_32.npz"), m=m, h_demag=kern.field(m),
                        h_eff=rhs.h_total_quiet(0.0, m), numpy=np.__version__, scipy=scipy.__version__)
    print("bench_32 ok")


def main():
    groups = sys.argv[1:]
    if groups:
        for gname in groups:
            {"spatial": spatial_bias_golden, "sp4_protocol": sp4_protocol_golden,
             "radix5": radix5_goldens, "bench32": bench32_golden}[gname]()
        return
    ALL = ("exchange", "anisotropy", "dmi")
    # tiny grids: every term, every boundary mode
    case("box_6x5x4_all", (6, 5, 4), (1e-9, 2e-9, 1.5e-9),
         dict(Ms=8e5, A=1.3e-11, Ku=5e4, eK=(0.3, 0.2, 1.0), D=1e-3, alpha=0.1),
         ALL, 1, bias=(1e4, -2e3, 5e3), demag=True, dt=2e-14, nsteps=10, mri_steps=4)
    case("box_6x5x4_neumann", (6, 5, 4), (1e-9, 2e-9, 1.5e-9),
         dict(Ms=8e5, A=1.3e-11, Ku=5e4, alpha=0.02),
         ("exchange", "anisotropy"), 2, bias=(1e4, 0.0, 0.0), demag=True, dt=2e-14, nsteps=10)
    case("box_6x5x4_periodic", (6, 5, 4), (2e-9, 2.5e-9, 3e-9),
         dict(Ms=8e5, A=1.3e-11, alpha=0.1), ("exchange",), 3, ghost_mode="periodic",
         dt=2e-14, nsteps=5)
    case("odd_9x7x3", (9, 7, 3), (2e-9, 2e-9, 2e-9),
         dict(Ms=8e5, A=1.3e-11, Ku=1e4, alpha=0.3), ("exchange", "anisotropy"), 4,
         bias=(0.0, 5e3, 0.0), demag=True, dt=2e-14, nsteps=5)
    case("film_4x4x1", (4, 4, 1), (2e-9, 2e-9, 2e-9),
         dict(Ms=8e5, A=1.3e-11, alpha=0.1), ("exchange",), 7, bias=(0.0, 0.0, 1e4),
         demag=True, dt=2.5e-14, nsteps=5, mri_steps=3)
    case("chain_8x1x1", (8, 1, 1), (2e-9, 1e-9, 3e-9),
         dict(Ms=8e5, A=1.3e-11, D=2e-3, alpha=0.2), ("exchange", "dmi"), 8,
         demag=True, dt=1e-14, nsteps=3)
    case("col_1x5x6", (1, 5, 6), (1.5e-9, 1e-9, 1e-9),
         dict(Ms=8e5, A=1.3e-11, alpha=0.2), ("exchange",), 9, demag=True, dt=1e-14, nsteps=3)
    case("spin_1x1x1", (1, 1, 1), (1e-9, 1e-9, 1e-9),
         dict(Ms=8e5, alpha=0.2), (), 10, bias=(0.0, 0.0, 7.9577e5), demag=True,
         dt=1e-13, nsteps=5)
    case("disk_16_dmi", (16, 16, 1), (1e-9, 1e-9, 0.25e-9),
         dict(A=16e-12, Ku=5.5e5, D=4.5e-3, alpha=1.0), ALL, 11, msmap=disk,
         dt=1e-14, nsteps=10, mri_steps=3)
    case("disk_16_dmi_demag", (16, 16, 2), (1e-9, 1e-9, 0.5e-9),
         dict(A=16e-12, Ku=5.5e5, D=4.5e-3, alpha=0.5), ALL, 12, msmap=disk, demag=True,
         dt=1e-14, nsteps=5)
    # BASELINE configs at their real sizes (packed tensor pinned by hash only)
    dx4 = 500e-9 / 128
    case("sp4_128x32x1", (128, 32, 1), (dx4, 125e-9 / 32, 3e-9),
         dict(Ms=8e5, A=1.3e-11, alpha=0.02), ("exchange",), 13,
         bias=(-19576.0, 3422.0, 0.0), demag=True, dt=3.125e-13 * 0.5, nsteps=20,
         store_tensor=False)
    lex = np.sqrt(1.3e-11 / (0.5 * 4e-7 * np.pi * 8e5 ** 2))
    dc = 8.47 * lex / 32
    case("sp3_32", (32, 32, 32), (dc, dc, dc),
         dict(Ms=8e5, A=1.3e-11, Ku=0.1 * 0.5 * 4e-7 * np.pi * 8e5 ** 2, eK=(0, 0, 1),
              alpha=0.5), ("exchange", "anisotropy"), 14, demag=True, dt=4e-14, nsteps=2,
         store_tensor=False)
    case("dmi_disk_100", (100, 100, 1), (1e-9, 1e-9, 0.25e-9),
         dict(A=16e-12, Ku=5.5e5, D=4.5e-3, alpha=1.0), ALL, 15, msmap=disk,
         dt=1e-14, nsteps=20)

    # known answers of the tensor itself
    kw = {}
    for i, cell in enumerate([(1, 1, 1), (2, 1, 1), (1, 2, 3), (10, 10, 1), (1, 1, 5)]):
        kw[f"self_{i}"] = rdemag.self_demag_tensor(*(c * 1e-9 for c in cell))
        kw[f"self_{i}_cell"] = np.array(cell, dtype=np.float64) * 1e-9
    kw["tensor_432"] = rdemag.tensor_elements(4, 3, 2, 1e-9, 2e-9, 1.5e-9)
    kw["tensor_chain120"] = rdemag.tensor_elements(120, 1, 1, 1e-9, 1e-9, 1e-9)
    np.savez_compressed(os.path.join(OUT, "tensor_known.npz"), **kw)

    # SP4 field-1 protocol trace: S-state-like start (+x with a tilt), 400 steps
    g = GridSpec(128, 32, 1, dx4, 125e-9 / 32, 3e-9)
    mat = MaterialMap(g, Ms=8e5, A=1.3e-11, alpha=0.02)
    kern = rdemag.DemagKernel.build(g)
    rhs = PartitionedRHS(mat, exchange=True, demag=kern,
                         bias=np.array([-19576.0, 3422.0, 0.0]))
    X, Y, _ = g.cell_centers()
    m = VectorField3(g)
    ang = 0.3 * np.sin(np.pi * X / (500e-9))
    m.data[0] = np.cos(ang) * 8e5
    m.data[1] = np.sin(ang) * 8e5
    m.data[2] = 0.01 * 8e5
    renormalize(m, mat)
    m0 = m.data.copy()
    dt = 3.125e-13 * 0.5  # stable_dt(3.90625e-9, ...) = 7.81e-14*... see bench/common.py
    from magnex.bench.common import stable_dt
    dt = stable_dt(g.dx, 1.3e-11, 8e5)
    st = SimState(VectorField3(g, m0.copy()))
    sim = Simulation(st, rhs, IntegratorSpec("rk4", dt), sample_every=10,
                     energy_in_samples=True)
    tr = sim.run_until(StopCondition(max_steps=400))
    np.savez_compressed(os.path.join(OUT, "sp4_trace.npz"), m0=m0, dt=dt,
                        t=tr.column("t"), mx=tr.column("mx"), my=tr.column("my"),
                        mz=tr.column("mz"), e_demag=tr.column("e_demag"),
                        e_exch=tr.column("e_exch"), e_total=tr.column("e_total"),
                        n_demag=tr.column("n_demag_evals"),
                        final_sha=sha(st.m.data), mean_final=mean_normalized(st.m, mat))
    print("sp4_trace ok, dt", dt, "final mean", mean_normalized(st.m, mat))
    radix5_goldens()
    spatial_bias_golden()
    sp4_protocol_golden()
    bench32_golden()


if __name__ == "__main__":
    main()
