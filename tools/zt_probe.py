import os, sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2602_12242_b200 as mx
case = sys.argv[1]
g = mx.GridSpec(512, 128, 64, 4e-9, 4e-9, 4e-9)
mat = mx.MaterialMap(g, Ms=8e5, A=1.3e-11, Ku=5e4, eK=(0, 0, 1), alpha=0.1)
m = mx.VectorField3(g, np.random.default_rng(1).standard_normal((3,) + g.shape)); mx.renormalize(m, mat)
if case == "heff_nodemag":
    r = mx.PartitionedRHS(mat, exchange=True, anisotropy=True)
    print(case, float(np.abs(r.h_total_quiet(0.0, m.data)).max()))
elif case == "rhs_demag":
    r = mx.PartitionedRHS(mat, exchange=True, demag=mx.DemagKernel.build(g, symmetric=True))
    print(case, float(np.abs(r.rhs_total(0.0, m.data)).max()))
elif case.startswith("run"):
    demag = case.endswith("demag")
    r = mx.PartitionedRHS(mat, exchange=True, demag=mx.DemagKernel.build(g, symmetric=True) if demag else None)
    st = mx.SimState(m.copy())
    mx.Simulation(st, r, mx.IntegratorSpec("rk4", 3e-14), sample_every=10**9, energy_in_samples=False).run_until(mx.StopCondition(max_steps=1))
    print(case, float(st.m.data.sum()))
