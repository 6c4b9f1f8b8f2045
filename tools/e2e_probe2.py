"""Per-call overhead of the device loop at 512^3: mxb_run with nsteps = 1 vs
nsteps = 10, eager (MXB_GRAPHS=0 in a second process) vs graph replay, and
mxb_state_mean."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import setup_problem  # noqa: E402
from paper_2602_12242_b200 import _lib as L  # noqa: E402
from paper_2602_12242_b200.llg import _ORDER  # noqa: E402

mx, g, mat, kern, rhs, m, dt, bias, tb = setup_problem(int(os.environ.get("N", "512")))
ctx = mat._ctx()
L.check(ctx.call("mxb_state_set", L.dptr(m.data)))
ts = rhs._terms_struct(tuple(x for x in _ORDER if x in rhs.enabled_terms()))
args = L.RunArgs()
args.method = L.RK4
args.dt = dt
args.eq_tol = -1.0
args.renorm_each_stage = 1
args.theta = 0.1
args.bias_vec = (C.c_double * 3)(*bias)
st = L.RunStats()


def run(n):
    args.nsteps = n
    L.check(ctx.call("mxb_run", kern._d.h, C.byref(ts), C.byref(args), C.byref(st)))


run(2)
tag = "graphs" if os.environ.get("MXB_GRAPHS", "1") != "0" else "eager"
for rep in range(2):
    t0 = time.perf_counter()
    for _ in range(10):
        run(1)
    t1 = time.perf_counter()
    run(10)
    t2 = time.perf_counter()
    mb = np.zeros(3)
    for _ in range(10):
        L.check(ctx.call("mxb_state_mean", L.dptr(mb)))
    t3 = time.perf_counter()
    print(f"[{tag}] 10 x mxb_run(1): {1e3*(t1-t0)/10:.2f} ms/step   mxb_run(10): {1e3*(t2-t1)/10:.2f} ms/step   "
          f"mxb_state_mean: {1e3*(t3-t2)/10:.2f} ms", flush=True)
