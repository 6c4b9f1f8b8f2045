"""Probe the plane pipeline on one shape: build, evaluate, time (one process per shape)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_12242_b200 as mx  # noqa: E402

nx, ny, nz = (int(v) for v in sys.argv[1:4])
g = mx.GridSpec(nx, ny, nz, 2e-9, 2e-9, 2e-9)
t0 = time.perf_counter()
k = mx.DemagKernel.build(g, symmetric=True)
tb = time.perf_counter() - t0
m = np.random.default_rng(1).normal(size=(3,) + g.shape)
h = k.field(m)
import ctypes as C  # noqa: E402
from paper_2602_12242_b200 import _lib as L  # noqa: E402
mat = mx.MaterialMap(g, Ms=8e5)
ctx = mat._ctx()
L.check(ctx.call("mxb_state_set", L.dptr(np.ascontiguousarray(m * 8e5))))
ms = C.c_double()
passes = np.zeros(5)
L.check(ctx.call("mxb_time_demag", k._d.h, 5, C.byref(ms), L.dptr(passes)))
print(f"dims={nx}x{ny}x{nz} pipe={os.environ.get('MXB_PIPE')} build={tb:.1f}s eval_ms={ms.value:.3f} "
      f"passes={np.round(passes, 3).tolist()} finite={bool(np.isfinite(h).all())}", flush=True)
