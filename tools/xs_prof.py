"""One RK4 step of the bench problem (512^3) through mxb_time_steps: a target
for ncu --kernel-name on the x-row fused stage or any kernel of the step."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
from bench import setup_problem  # noqa: E402
from paper_2602_12242_b200 import _lib as L  # noqa: E402
from paper_2602_12242_b200.llg import _ORDER  # noqa: E402

mx, g, mat, kern, rhs, m, dt, bias, _ = setup_problem(int(sys.argv[1]) if len(sys.argv) > 1 else 512)
ctx = mat._ctx()
L.check(ctx.call("mxb_state_set", L.dptr(m.data)))
ts = rhs._terms_struct(tuple(x for x in _ORDER if x in rhs.enabled_terms()))
ms, nl = C.c_double(), C.c_int64()
L.check(ctx.call("mxb_time_steps", kern._d.h, C.byref(ts), dt, 2, L.dptr(np.ascontiguousarray(bias)),
                 C.byref(ms), None, C.byref(nl)))
print("ms per step", ms.value / 2, "launches", nl.value)
