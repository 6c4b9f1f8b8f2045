"""FNO surrogate inference time on one B200 vs the CPU oracle (width 32, modes 12).

  python tools/bench_fno.py
Prints one JSON line per film size.  GPU time includes the host<->device copies
(FnoDemag.field semantics); the device-only time uses mxb_fno_infer_dev.
"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from oracle import fno_oracle as FO  # noqa: E402
from paper_2602_12242_b200 import _lib as L  # noqa: E402
from paper_2602_12242_b200 import fno as F  # noqa: E402
from tests.fno_tables import tensors  # noqa: E402

t = tensors(32, (12, 12), 23)
model = F.FnoModel.from_tensors(t).freeze()
for H, W in ((32, 128), (128, 128), (512, 512), (2048, 2048)):
    x = np.random.default_rng(0).standard_normal((3, H, W))
    model.infer(x)
    n = 20 if H * W <= 512 * 512 else 5
    t0 = time.perf_counter()
    for _ in range(n):
        y = model.infer(x)
    host_ms = (time.perf_counter() - t0) / n * 1e3
    dx = torch.from_numpy(x).cuda()
    dy = torch.empty_like(dx)
    h = model._device(H, W).h
    L.check(L.load().mxb_fno_infer_dev(h, C.c_void_p(dx.data_ptr()), C.c_void_p(dy.data_ptr())))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        L.load().mxb_fno_infer_dev(h, C.c_void_p(dx.data_ptr()), C.c_void_p(dy.data_ptr()))
    torch.cuda.synchronize()
    dev_ms = (time.perf_counter() - t0) / n * 1e3
    cpu_ms = None
    if H * W <= 512 * 512:
        f = FO.as_f64(t)
        t0 = time.perf_counter()
        ref = FO.infer(f, x)
        cpu_ms = (time.perf_counter() - t0) * 1e3
        err = float(np.max(np.abs(y - ref)) / np.max(np.abs(ref)))
    else:
        err = None
    print(json.dumps({"fno": f"{H}x{W} width 32 modes 12", "gpu_ms_e2e": host_ms, "gpu_ms_device": dev_ms,
                      "cpu_oracle_ms": cpu_ms, "rel_err_vs_oracle": err}), flush=True)
