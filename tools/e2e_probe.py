"""Where the end-to-end time of Simulation.run_until goes at 512^3 (one B200)."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import setup_problem  # noqa: E402
from paper_2602_12242_b200 import _lib as L  # noqa: E402

mx, g, mat, kern, rhs, m, dt, bias, tb = setup_problem(512)
N = g.n_cells
pinned = C.c_void_p()
L.check(L.load().mxb_host_alloc(m.data.nbytes, C.byref(pinned)))
host = np.ctypeslib.as_array((C.c_double * (3 * N)).from_address(pinned.value)).reshape(m.data.shape)
host[...] = m.data
ctx = mat._ctx()
import torch  # noqa: E402
for rep in range(2):
    t0 = time.perf_counter()
    L.check(ctx.call("mxb_state_set", L.dptr(host)))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    buf = np.empty_like(host)
    L.check(ctx.call("mxb_state_get", L.dptr(buf)))
    t2 = time.perf_counter()
    L.check(ctx.call("mxb_state_get", L.dptr(buf)))
    t3 = time.perf_counter()
    print(f"state_set(pinned) {1e3*(t1-t0):.1f} ms  state_get(fresh pageable) {1e3*(t2-t1):.1f} ms  "
          f"state_get(touched pageable) {1e3*(t3-t2):.1f} ms", flush=True)
for chunk in (1, 10):
    st = mx.SimState(mx.VectorField3(g, host))
    sim = mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", dt), sample_every=1, energy_in_samples=False)
    sim.CHUNK = chunk
    t0 = time.perf_counter()
    sim.run_until(mx.StopCondition(max_steps=10))
    el = time.perf_counter() - t0
    print(f"run_until 10 steps CHUNK={chunk}: {1e3*el:.0f} ms -> {N*10/el:.3e} cell-steps/s", flush=True)
if "--profile" in sys.argv:
    import cProfile
    import pstats
    st = mx.SimState(mx.VectorField3(g, host))
    sim = mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", dt), sample_every=1, energy_in_samples=False)
    sim.CHUNK = 1
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    sim.run_until(mx.StopCondition(max_steps=20))
    pr.disable()
    el = time.perf_counter() - t0
    print(f"profiled run_until 20 steps: {1e3*el:.0f} ms -> {N*20/el:.3e}", flush=True)
    pstats.Stats(pr).sort_stats("tottime").print_stats(14)
