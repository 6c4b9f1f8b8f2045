"""Time-to-solution of the BASELINE.json configs through the public API
(Simulation.run_until from host state, i.e. end to end), on one B200.

  python tools/bench_configs.py [--quick]

Prints one JSON line per config.  Tensor builds are excluded (reported
separately), as in the reference's own timing convention.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2602_12242_b200 as mx  # noqa: E402


def timed_run(sim, stop):
    import torch
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tr = sim.run_until(stop)
    return time.perf_counter() - t0, tr


def stable_dt(dx, A, Ms, safety=0.5):
    return safety * 2.5e-14 * (dx / 0.78125e-9) ** 2 * ((1.3e-11 / 8e5) / (A / Ms))


def sp4(quick):
    """µMAG SP4 field 1 on 128x32x1 (500x125x3 nm), RK4 at stable_dt, energies every ~1 ps."""
    g = mx.GridSpec(128, 32, 1, 500e-9 / 128, 125e-9 / 32, 3e-9)
    mat = mx.MaterialMap(g, Ms=8e5, A=1.3e-11, alpha=0.02)
    t0 = time.perf_counter()
    k = mx.DemagKernel.build(g)
    tb = time.perf_counter() - t0
    rhs = mx.PartitionedRHS(mat, exchange=True, demag=k, bias=(-19576.0, 3422.0, 0.0))
    m = mx.VectorField3.from_uniform(g, (8e5, 0.0, 0.0))
    m.data[1] += 1e3
    mx.renormalize(m, mat)
    dt = stable_dt(g.dx, 1.3e-11, 8e5)
    st = mx.SimState(m)
    every = max(1, round(1e-12 / dt))
    sim = mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", dt), sample_every=every,
                        energy_in_samples=True)
    T = 0.2e-9 if quick else 2e-9
    el, tr = timed_run(sim, mx.StopCondition(max_time=T))
    n = st.step
    return {"config": "SP4 128x32x1 field-1 RK4 (energies in samples)", "sim_time_s": T,
            "steps": n, "wall_s": el, "steps_per_s": n / el, "cell_steps_per_s": g.n_cells * n / el,
            "samples": len(tr.samples), "tensor_build_s": tb,
            "cpu_reference_wall_s_for_2ns": 55.7}


def table2(method):
    """Paper Table II setup: SP4 at 0.78125 nm = 640x160x4, exchange + demag + bias,
    RK4 5 steps of 2.5e-14 s, or MRI 1 step of 1.25e-13 s."""
    d = 0.78125e-9
    g = mx.GridSpec(640, 160, 4, d, d, d)
    mat = mx.MaterialMap(g, Ms=8e5, A=1.3e-11, alpha=0.02)
    t0 = time.perf_counter()
    k = mx.DemagKernel.build(g)
    tb = time.perf_counter() - t0
    rhs = mx.PartitionedRHS(mat, exchange=True, demag=k, bias=(-19576.0, 3422.0, 0.0))
    rng = np.random.default_rng(3)
    m = mx.VectorField3(g, rng.normal(size=(3,) + g.shape) * 0.05 + np.array([1.0, 0.3, 0.0])[:, None, None, None])
    mx.renormalize(m, mat)
    if method == "rk4":
        spec = mx.IntegratorSpec("rk4", 2.5e-14)
    else:
        spec = mx.IntegratorSpec("mri-kw3", 1.25e-13, theta=0.1)
    # warm-up on a copy, then time the 1.25e-13 s interval
    st = mx.SimState(m.copy())
    mx.Simulation(st, rhs, spec, sample_every=10 ** 9, energy_in_samples=False).run_until(
        mx.StopCondition(max_steps=1))
    st = mx.SimState(m.copy())
    sim = mx.Simulation(st, rhs, spec, sample_every=10 ** 9, energy_in_samples=False)
    el, tr = timed_run(sim, mx.StopCondition(max_time=1.25e-13))
    paper = 0.133 if method == "rk4" else 0.069
    return {"config": f"Table II 640x160x4 {method} over 1.25e-13 s", "steps": st.step,
            "wall_s": el, "cell_steps_per_s": g.n_cells * st.step / el,
            "paper_gv100_s": paper, "speedup_vs_paper_gv100": paper / el,
            "counters": tr.counters, "tensor_build_s": tb}


def sp3(quick):
    """µMAG SP3 cube 32^3 at L = 8.47 lex: exchange + uniaxial anisotropy + demag, RK4."""
    lex = np.sqrt(1.3e-11 / (0.5 * mx.MU0 * 8e5 ** 2))
    dc = 8.47 * lex / 32
    g = mx.GridSpec(32, 32, 32, dc, dc, dc)
    Km = 0.5 * mx.MU0 * 8e5 ** 2
    mat = mx.MaterialMap(g, Ms=8e5, A=1.3e-11, Ku=0.1 * Km, eK=(0, 0, 1), alpha=0.5)
    k = mx.DemagKernel.build(g)
    rhs = mx.PartitionedRHS(mat, exchange=True, anisotropy=True, demag=k)
    m = mx.VectorField3.from_uniform(g, (0.0, 0.1, 1.0))
    mx.renormalize(m, mat)
    dt = stable_dt(dc, 1.3e-11, 8e5)
    n = 200 if quick else 2000
    st = mx.SimState(m)
    sim = mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", dt), sample_every=10 ** 9,
                        energy_in_samples=False)
    el, _ = timed_run(sim, mx.StopCondition(max_steps=n))
    return {"config": "SP3 32^3 exchange+anisotropy+demag RK4", "steps": n, "wall_s": el,
            "steps_per_s": n / el, "cell_steps_per_s": g.n_cells * n / el,
            "cpu_reference_s_per_step": 0.124}


def disk(quick):
    """Interfacial-DMI nanodot 100x100x1 (R = 50 nm, dx = 1 nm), exchange + anisotropy + DMI,
    relaxation with alpha = 1 (bench/skyrmion.py:61-132 at dx = 1 nm)."""
    g = mx.GridSpec(100, 100, 1, 1e-9, 1e-9, 0.25e-9)
    X, Y, _ = g.cell_centers()
    inside = (X - 50e-9) ** 2 + (Y - 50e-9) ** 2 <= (50e-9) ** 2
    mat = mx.MaterialMap(g, Ms=np.where(inside, 1.1e6, 0.0), A=16e-12, Ku=5.5e5, eK=(0, 0, 1),
                         D=4.5e-3, alpha=1.0)
    rhs = mx.PartitionedRHS(mat, exchange=True, anisotropy=True, dmi=True)
    r = np.sqrt((X - 50e-9) ** 2 + (Y - 50e-9) ** 2)
    th = np.pi * np.clip(1 - r / 50e-9, 0, 1)
    m = mx.VectorField3(g, np.stack([np.sin(th) * (X - 50e-9) / np.maximum(r, 1e-30),
                                     np.sin(th) * (Y - 50e-9) / np.maximum(r, 1e-30),
                                     np.cos(th)]) * mat.Ms)
    mx.renormalize(m, mat)
    dt = stable_dt(1e-9, 16e-12, 1.1e6)
    n = 500 if quick else 5000
    st = mx.SimState(m)
    sim = mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", dt), sample_every=10 ** 9,
                        energy_in_samples=False)
    el, _ = timed_run(sim, mx.StopCondition(max_steps=n))
    return {"config": "DMI disk 100x100x1 RK4 (no demag, as the reference suite)", "steps": n,
            "wall_s": el, "steps_per_s": n / el, "cell_steps_per_s": g.n_cells * n / el,
            "cpu_reference_s_per_step": 0.0241}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    for f in (lambda: sp4(a.quick), lambda: table2("rk4"), lambda: table2("mri"),
              lambda: sp3(a.quick), lambda: disk(a.quick)):
        print(json.dumps(f()), flush=True)


if __name__ == "__main__":
    main()
