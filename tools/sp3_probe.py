"""SP3-sized step (32^3, exchange + anisotropy + demag, RK4) for an ncu launch
list: how much of a launch-bound step is kernel time."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_12242_b200 as mx  # noqa: E402

g = mx.GridSpec(32, 32, 32, 1e-8 / 32 * 10, 1e-8 / 32 * 10, 1e-8 / 32 * 10)
mat = mx.MaterialMap(g, Ms=1e6, A=1e-11, Ku=1e5, eK=(0, 0, 1), alpha=0.5)
m = mx.VectorField3(g, np.random.default_rng(0).standard_normal((3,) + g.shape))
mx.renormalize(m, mat)
rhs = mx.PartitionedRHS(mat, exchange=True, anisotropy=True, demag=mx.DemagKernel.build(g))
st = mx.SimState(m)
sim = mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", 1e-14), sample_every=10 ** 9, energy_in_samples=False)
sim.run_until(mx.StopCondition(max_steps=int(sys.argv[1]) if len(sys.argv) > 1 else 4))
print("ok")
