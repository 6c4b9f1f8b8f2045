"""The BASELINE thin-film config (2048 x 2048 x 64, 4 nm cells, permalloy,
demag + exchange + bias) on one B200: tensor build, one demag
evaluation and RK4 steps through the public API (not a bench: wall clocks)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_12242_b200 as mx  # noqa: E402

nx, ny, nz = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (2048, 2048, 64)))
g = mx.GridSpec(nx, ny, nz, 4e-9, 4e-9, 4e-9)
mat = mx.MaterialMap(g, Ms=8e5, A=1.3e-11, alpha=0.02)
t0 = time.perf_counter()
kern = mx.DemagKernel.build(g, symmetric=True)
tb = time.perf_counter() - t0
print(f"grid {nx}x{ny}x{nz} padded {kern.padded} pipeline={kern.pipeline} build {tb:.1f} s", flush=True)
rng = np.random.default_rng(0)
m = np.zeros((3,) + g.shape)
m[0] = 1.0
m += 0.01 * rng.standard_normal(m.shape)
m = mx.VectorField3(g, m)
mx.renormalize(m, mat)
t0 = time.perf_counter()
h = kern.field(m.data)
print(f"first field {time.perf_counter() - t0:.2f} s, finite {bool(np.isfinite(h).all())}", flush=True)
del h
rhs = mx.PartitionedRHS(mat, exchange=True, demag=kern, bias=(1e4, 0.0, 0.0))
dt = 0.1 * 4e-9 ** 2 * 8e5 * mx.MU0 / (2 * 1.3e-11) / abs(mx.GAMMA) if hasattr(mx, "GAMMA") else 1e-14
st = mx.SimState(m)
sim = mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", 1e-14), sample_every=10 ** 9, energy_in_samples=False)
sim.run_until(mx.StopCondition(max_steps=1))
for steps in (5, 10):
    t0 = time.perf_counter()
    sim.run_until(mx.StopCondition(max_steps=steps))
    el = time.perf_counter() - t0
    print(f"{steps} RK4 steps {el:.2f} s -> {g.n_cells * steps / el:.3e} cell-steps/s (wall, incl. state up/download)",
          flush=True)
