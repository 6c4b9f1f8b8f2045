"""Small driver for ncu: builds the synthetic workload at n^3 and runs a few
RK4 steps (plus demag evaluations) so each kernel of the hot path launches a
handful of times.  Not a benchmark (timings under ncu are not valid)."""
import argparse
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from bench import setup_problem  # noqa: E402
from paper_2602_12242_b200 import _lib as L  # noqa: E402
from paper_2602_12242_b200.llg import _ORDER  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--steps", type=int, default=2)
    a = ap.parse_args()
    mx, g, mat, kern, rhs, m, dt, bias, _ = setup_problem(a.n)
    ctx = mat._ctx()
    L.check(ctx.call("mxb_state_set", L.dptr(m.data)))
    ts = rhs._terms_struct(tuple(x for x in _ORDER if x in rhs.enabled_terms()))
    b = np.ascontiguousarray(bias)
    t, s = C.c_double(), C.c_double()
    nl = C.c_int64()
    L.check(ctx.call("mxb_time_steps", kern._d.h, C.byref(ts), dt, a.steps, L.dptr(b),
                     C.byref(t), None, C.byref(nl)))
    print("ok", t.value)


if __name__ == "__main__":
    main()
