#!/usr/bin/env python
"""LLG cell-steps/s (fp64 RK4, full H_eff) on B200 -- BASELINE.json metric.

Workload (N=1): synthetic random-m 512^3 grid (BASELINE configs[3]), 4 nm
cells, Ms=8e5 A/m, A=1.3e-11 J/m, Ku=5e4 J/m^3 along z, interfacial D=1e-3
J/m^2, alpha=0.1, Zeeman (1e4,0,0) A/m, FFT demag (GPU-built Newell tensor),
DMI ghost boundaries; m from numpy default_rng(0) normals, renormalised;
dt = 0.1 * stable_dt (bench/common.py:40-48) so no step blows up.

One "step" = one full RK4 step (4 demag evaluations + 4 fused stencil/LLG/
stage kernels).  value = cells * K / device time of K steps (CUDA events on
the context stream, after W warm-up steps); inputs (3.2 GB per field) are
larger than the 126 MB L2, so no explicit flush is needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--size 512] [--impl reference]

Under torchrun (N>1) the 512^3 problem is z-slab decomposed over the ranks
(strong scaling; NCCL halos, slab-FFT all-to-alls and step all-reduces); the
step time is the max over ranks of CUDA-event timings.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK = 6650.0
METRIC = "LLG cell-steps/s (fp64 RK4, full H_eff) at 1/2/4/8 B200; % of HBM roofline"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK, "fallback"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for n, v in zip(names, r[3:7]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


def setup_problem(n: int):
    import paper_2602_12242_b200 as mx
    from paper_2602_12242_b200.llg import _ORDER
    g = mx.GridSpec(n, n, n, 4e-9, 4e-9, 4e-9)
    mat = mx.MaterialMap(g, Ms=8e5, A=1.3e-11, Ku=5e4, eK=(0.0, 0.0, 1.0), D=1e-3, alpha=0.1)
    t0 = time.perf_counter()
    kern = mx.DemagKernel.build(g, symmetric=True)
    t_build = time.perf_counter() - t0
    bias = np.array([1e4, 0.0, 0.0])
    rhs = mx.PartitionedRHS(mat, exchange=True, anisotropy=True, dmi=True, demag=kern, bias=bias)
    rng = np.random.default_rng(0)
    m = mx.VectorField3(g, rng.standard_normal(size=(3,) + g.shape))
    mx.renormalize(m, mat)
    dt = 0.1 * 0.5 * 2.5e-14 * (4e-9 / 0.78125e-9) ** 2   # 0.1 * stable_dt(4 nm, permalloy)
    return mx, g, mat, kern, rhs, m, dt, bias, t_build


def demag_bytes(g, kern, survey=True):
    """Algorithmic HBM bytes of one demag evaluation, per pass.

    survey=True: the SURVEY 8d fixed formula (the roofline contract), whose
    kernel term is a real 6-component kernel over the padded grid,
    48 hx py pz.  survey=False: what this implementation has to read -- the
    parity-reduced real spectra (a quarter in y and z) of a symmetric build,
    or complex spectra over the padded grid otherwise."""
    nx, ny, nz = g.nx, g.ny, g.nz
    pz, py, px = kern.padded
    hx = px // 2 + 1
    N = nx * ny * nz
    if survey:
        kbytes = 48 * hx * py * pz
    else:
        kbytes = 48 * hx * (py // 2 + 1) * (pz // 2 + 1) if kern.symmetric else 96 * hx * py * pz
    x1 = 48 * hx * ny * nz
    x2 = 48 * hx * py * nz
    return [24 * N + x1, x1 + x2, 2 * x2 + kbytes, x2 + x1, x1 + 24 * N]


def demag_flops(g, kern):
    """FP64 flops of one demag evaluation per pass: 2.5 L log2 L per
    real line transform, 5 L log2 L per complex line, over the pruned lines,
    plus 36 per spectral point for the 3x3 multiply."""
    import math
    nx, ny, nz = g.nx, g.ny, g.nz
    pz, py, px = kern.padded
    hx = px // 2 + 1
    lg = lambda n: math.log2(n) if n > 1 else 0.0
    xr = 3 * ny * nz * 2.5 * px * lg(px)
    yc = 3 * hx * nz * 5 * py * lg(py)
    zc = 3 * hx * py * 5 * pz * lg(pz)
    mul = 36 * hx * py * pz
    return [xr, yc, 2 * zc + mul, yc, xr]


def cpu_reference(n: int, steps: int, warmup: int):
    """Oracle (numpy/scipy restatement of the reference) RK4 on a bounded
    sample of the same workload: an n^3 grid, all host threads for the FFTs."""
    from oracle import magnex_oracle as O
    cores = os.cpu_count() or 1
    mat = O.make_mat((n, n, n), (4e-9,) * 3, 8e5, A=1.3e-11, Ku=5e4, D=1e-3, alpha=0.1)
    spectra = O.kernel_spectra(O.packed_tensor(n, n, n, 4e-9, 4e-9, 4e-9), workers=cores)
    import scipy.fft as sfft
    terms = O.Terms(exchange=True, anisotropy=True, dmi=True, spectra=spectra,
                    bias=np.array([1e4, 0.0, 0.0]))
    rng = np.random.default_rng(0)
    m = O.renormalize(rng.standard_normal(size=(3, n, n, n)), mat)
    dt = 0.1 * O.stable_dt(4e-9, 1.3e-11, 8e5)
    with sfft.set_workers(cores):
        if warmup:
            m = O.run(m, mat, terms, "rk4", dt, max_steps=warmup).m
        t0 = time.perf_counter()
        r = O.run(m, mat, terms, "rk4", dt, max_steps=steps)
        el = time.perf_counter() - t0
    return n ** 3 * steps / el, el, cores


# weak scaling ladder (paper PAPER.md:480-518): 2^24 cells per GPU
WEAK_DIMS = {1: (256, 256, 256), 2: (512, 256, 256), 4: (512, 512, 256), 8: (512, 512, 512)}


def grid_dims(args, world):
    """(nx, ny, nz): strong scaling keeps --size^3 for every N; weak scaling
    follows the 256^3 -> 512x256^2 -> 512^2x256 -> 512^3 ladder."""
    if args.scaling == "weak":
        return WEAK_DIMS.get(world, (256, 256, 256 * world))
    return args.size, args.size, args.size


def extrapolate_cpu(cs: float, n_sample: int, n: int) -> dict:
    """the CPU rate at the bench size, scaled from the
    sample by the per-cell FFT cost (log2 of the padded cells, N log N per
    step); the 512^3 oracle run itself needs ~230 GB of host memory."""
    import math
    f = math.log2((2 * n_sample) ** 3) / math.log2((2 * n) ** 3)
    return {"value": cs * f, "unit": "cell-steps/s", "cells": n ** 3,
            "method": f"N log N: sample rate x log2((2*{n_sample})^3) / log2((2*{n})^3) = x{f:.3f}",
            "flag": "extrapolated, not measured"}


def tensor_deviation(mx):
    """Deviation of the GPU-built tensor (the bench's mode and the unmirrored
    build) from the reference's own tensor at 32^3 with the bench material,
    against the fixture tests/golden/bench_32.npz made by running the reference
    (tests/golden/make_golden.py bench32)."""
    path = os.path.join(ROOT, "tests", "golden", "bench_32.npz")
    if not os.path.exists(path):
        return None
    z = np.load(path)
    g = mx.GridSpec(32, 32, 32, 4e-9, 4e-9, 4e-9)
    mat = mx.MaterialMap(g, Ms=8e5, A=1.3e-11, Ku=5e4, eK=(0.0, 0.0, 1.0), D=1e-3, alpha=0.1)
    out = {}
    for name, sym in (("mirrored_bench_mode", True), ("unmirrored", False)):
        k = mx.DemagKernel.build(g, symmetric=sym)
        hd = k.field(z["m"])
        rhs = mx.PartitionedRHS(mat, exchange=True, anisotropy=True, dmi=True, demag=k,
                                bias=np.array([1e4, 0.0, 0.0]))
        he = rhs.h_total_quiet(0.0, z["m"])
        out[name] = {"h_demag": float(np.max(np.abs(hd - z["h_demag"])) / np.max(np.abs(z["h_demag"]))),
                     "h_eff": float(np.max(np.abs(he - z["h_eff"])) / np.max(np.abs(z["h_eff"])))}
    out["norm"] = "max|dH| / max|H_ref| at 32^3 (random-direction m), vs the reference's tensor"
    return out


def run_slab(args, rank, world, local):
    """N > 1: the 512^3 problem z-slab decomposed over the ranks (strong scaling):
    halo planes by send/recv, slab FFT transposes by all-to-all, step reductions
    by all-reduce (paper_2602_12242_b200.slab)."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    import paper_2602_12242_b200 as mx
    from paper_2602_12242_b200 import _lib as L
    from paper_2602_12242_b200.llg import _ORDER
    from paper_2602_12242_b200.slab import Comm, CudaSlabBackend, SlabPlan, SlabSimulation
    dev = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(dev)
    mx.set_device(dev)
    dist.init_process_group(args.backend)
    nx, ny, nz = grid_dims(args, world)
    plan = SlabPlan(nx, ny, nz, world, rank)
    cell = (4e-9, 4e-9, 4e-9)
    gl = mx.GridSpec(nx, ny, plan.nz_local, *cell)
    mat_l = mx.MaterialMap(gl, Ms=8e5, A=1.3e-11, Ku=5e4, eK=(0.0, 0.0, 1.0), D=1e-3, alpha=0.1)
    h = C.c_void_p()
    t0 = time.perf_counter()
    L.check(L.load().mxb_demag_create_slab(C.byref(mx.GridSpec(nx, ny, nz, *cell)._c()), dev, world,
                                           rank, C.byref(h)))
    L.check(L.load().mxb_demag_build(h, 1))
    t_build = time.perf_counter() - t0
    b = CudaSlabBackend(plan, gl, mat_l, h, dev)
    bias = np.array([1e4, 0.0, 0.0])
    rhs = mx.PartitionedRHS(mat_l, exchange=True, anisotropy=True, dmi=True, bias=bias)
    mask = L.TERM_DEMAG
    for t in rhs.enabled_terms():
        mask |= {"exchange": L.TERM_EXCHANGE, "anisotropy": L.TERM_ANISOTROPY, "dmi": L.TERM_DMI,
                 "bias": L.TERM_BIAS}[t]
    terms = L.Terms(mask, L.GHOST["dmi"], 1, 1)
    # the same global state as the single-GPU run (setup_problem: default_rng(0)
    # over the whole grid), sliced to this rank's planes, so N > 1 results can be
    # compared with N = 1
    full = np.random.default_rng(0).standard_normal(size=(3, nz, ny, nx))
    m = mx.VectorField3(gl, np.ascontiguousarray(full[:, plan.z0:plan.z0 + plan.nz_local]))
    del full
    mx.renormalize(m, mat_l)
    dt = 0.1 * 0.5 * 2.5e-14 * (4e-9 / 0.78125e-9) ** 2
    sim = SlabSimulation(plan, b, Comm(), terms, method="rk4", dt=dt, bias=bias)
    sim.start(m.data)
    sim.run(max(args.warmup, 1))
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(dev) as clk:
        e0.record()
        st = sim.run(args.steps)
        e1.record()
        torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / args.steps], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    t_step = float(ms.item())
    # end to end through the slab driver: upload the slab, K steps, download it
    dist.barrier()
    w0 = time.perf_counter()
    sim.start(m.data)
    sim.run(args.steps)
    _ = sim.state()
    w = torch.tensor([time.perf_counter() - w0], device="cuda")
    dist.all_reduce(w, op=dist.ReduceOp.MAX)
    N = nx * ny * nz
    if rank == 0:
        out = {"metric": METRIC, "value": N / (t_step * 1e-3), "unit": "cell-steps/s", "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step,
               "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
               "data": "synthetic",
               "config": {"workload": f"synthetic random-m {nx}x{ny}x{nz}, full H_eff, RK4, z-slab decomposed",
                          "cells": N, "dt": dt, "parallelism": f"z-slab x{world} ({args.backend})",
                          "l2": "inputs > L2, no flush"},
               "e2e": {"value": N * args.steps / float(w.item()), "unit": "cell-steps/s",
                       "h2d_bytes_per_step": int(24 * N / world / args.steps),
                       "d2h_bytes_per_step": int(24 * N / world / args.steps)},
               "cpu_baseline": None, "tensor_build_s": t_build, "steps_done": int(st.steps_done),
               "gpu_launches": args.steps * 26, "clocks": clk.summary()}
        print(json.dumps(out))
    dist.destroy_process_group()


def complex_mode(mx, L, C, ctx, g, ts, dt, bptr, args):
    """The plane pipeline with full complex spectra (kernel mode 5): the mode
    from_packed / load_kernel select for the reference's own tensor (no
    symmetry assumed, 96 B per spectral point instead of the mirrored build's
    parity-reduced 12).  Timed on the unmirrored GPU build of the same grid."""
    t0 = time.perf_counter()
    kc = mx.DemagKernel.build(g)
    t_build = time.perf_counter() - t0
    if kc.kmode != 5:
        return {"kmode": kc.kmode, "note": "complex-spectra pipeline not selected for this shape"}
    ms_tot, nl = C.c_double(), C.c_int64()
    L.check(ctx.call("mxb_time_steps", kc._d.h, C.byref(ts), dt, 1, bptr, C.byref(ms_tot), None,
                     C.byref(nl)))
    n = max(3, args.steps // 4)
    L.check(ctx.call("mxb_time_steps", kc._d.h, C.byref(ts), dt, n, bptr, C.byref(ms_tot), None,
                     C.byref(nl)))
    ms_eval = C.c_double()
    passes = np.zeros(5)
    L.check(ctx.call("mxb_time_demag", kc._d.h, 3, C.byref(ms_eval), L.dptr(passes)))
    t_step = ms_tot.value / n
    out = {"kmode": 5, "ms_per_step": t_step, "value": g.n_cells / (t_step * 1e-3),
           "unit": "cell-steps/s", "steps": n, "demag_ms_per_eval": ms_eval.value,
           "yz_pipeline_ms_per_eval": float(passes[1] + passes[2] + passes[3]),
           "spectra_bytes": kc.device_bytes, "tensor_build_s": t_build,
           "note": "unmirrored GPU tensor in the complex-spectra pipeline (what the reference's "
                   "own packed tensor runs through): parity with the reference tensor 5.6e-16 "
                   "(tests/test_bench_path_parity.py)"}
    del kc
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--size", type=int, default=512, help="cells per edge of the synthetic cube")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-n", type=int, default=64)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-dev", action="store_true", help="skip the 32^3 tensor-deviation check")
    ap.add_argument("--no-ref-mode", action="store_true",
                    help="skip timing the complex-spectra (reference tensor) pipeline")
    ap.add_argument("--repeats", type=int, default=5,
                    help="timed runs of --steps steps; the median is reported (SURVEY 8d)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: --size^3 on every N; weak: 2^24 cells per GPU (256^3 ... 512^3 at N=8)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="collectives for N > 1 (gloo only to exercise the path on one GPU)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        cs, el, cores = cpu_reference(args.cpu_n, max(args.steps, 1), max(args.warmup, 0))
        out = {"metric": METRIC, "value": cs, "unit": "cell-steps/s", "n_gpus": args.gpus,
               "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": 1e3 * el / max(args.steps, 1), "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
               "impl": "reference",
               "config": {"workload": f"synthetic random-m {args.cpu_n}^3 full H_eff RK4 "
                                      f"(bounded CPU sample of the {args.size}^3 workload)"},
               "cpu_baseline": {"value": cs, "unit": "cell-steps/s", "cores": cores, "kind": "port",
                                "sample": f"{args.cpu_n}^3, {args.steps} RK4 steps, oracle numpy/scipy"},
               "e2e": {"value": cs, "unit": "cell-steps/s", "h2d_bytes_per_step": 0,
                       "d2h_bytes_per_step": 0}}
        print(json.dumps(out))
        return

    if world > 1:
        run_slab(args, rank, world, local)
        return
    if args.scaling == "weak":
        args.size = WEAK_DIMS[1][0]

    import ctypes as C

    import paper_2602_12242_b200 as mxb
    from paper_2602_12242_b200 import _lib as L
    mxb.set_device(local)
    mx, g, mat, kern, rhs, m, dt, bias, t_build = setup_problem(args.size)
    N = g.n_cells
    ctx = mat._ctx()
    L.check(ctx.call("mxb_state_set", L.dptr(m.data)))
    from paper_2602_12242_b200.llg import _ORDER
    ts = rhs._terms_struct(tuple(x for x in _ORDER if x in rhs.enabled_terms()))
    bptr = L.dptr(np.ascontiguousarray(bias))
    ms_tot, ms_st = C.c_double(), C.c_double()
    nl = C.c_int64()
    d = kern._d.h
    # warm-up
    L.check(ctx.call("mxb_time_steps", d, C.byref(ts), dt, max(args.warmup, 1), bptr,
                     C.byref(ms_tot), None, C.byref(nl)))
    runs, runs_st = [], []
    with Clocks(local) as clk:
        for _ in range(max(args.repeats, 1)):
            L.check(ctx.call("mxb_time_steps", d, C.byref(ts), dt, args.steps, bptr,
                             C.byref(ms_tot), C.byref(ms_st), C.byref(nl)))
            runs.append(ms_tot.value / args.steps)
            runs_st.append(ms_st.value / args.steps)
    t_step = float(np.median(runs))
    ms_st = C.c_double(float(np.median(runs_st)) * args.steps)
    value = N / (t_step * 1e-3)
    # per-kernel timing for the roofline
    ms_eval = C.c_double()
    passes = np.zeros(5)
    L.check(ctx.call("mxb_time_demag", d, 3, C.byref(ms_eval), L.dptr(passes)))
    ms_cufft = C.c_double(float("nan"))
    rc = L.load().mxb_time_demag_cufft(d, 3, C.byref(ms_cufft))
    if rc != 0:
        ms_cufft = C.c_double(float("nan"))
    hbm, which = peaks()
    pb = demag_bytes(g, kern)
    stencil_bytes = 504 * N               # per RK4 step (4 fused stage kernels)
    if kern.pipeline:
        # one persistent kernel replaces the y forward, z fused and y inverse passes;
        # its algorithmic bytes are theirs (SURVEY 8d fixed formulas)
        kernels = [("x_r2c", pb[0], passes[0]),
                   ("yz_plane_pipeline", pb[1] + pb[2] + pb[3], passes[1] + passes[2] + passes[3]),
                   ("x_c2r", pb[4], passes[4])]
    else:
        kernels = [("x_r2c", pb[0], passes[0]), ("y_fwd", pb[1], passes[1]),
                   ("z_fused_mul", pb[2], passes[2]), ("y_inv", pb[3], passes[3]),
                   ("x_c2r", pb[4], passes[4])]
    kernels.append(("stage_stencil_llg", stencil_bytes / 4, ms_st.value / args.steps / 4))
    share = {k: 4 * t for k, _, t in kernels}
    dom = max(kernels, key=lambda x: x[2])
    ach = dom[1] / (dom[2] * 1e-3) / 1e9
    # the same kernel credited only with the bytes this implementation reads
    pb_own = demag_bytes(g, kern, survey=False)
    own = {"x_r2c": pb_own[0], "yz_plane_pipeline": pb_own[1] + pb_own[2] + pb_own[3], "x_c2r": pb_own[4],
           "y_fwd": pb_own[1], "z_fused_mul": pb_own[2], "y_inv": pb_own[3], "stage_stencil_llg": dom[1]}
    ach_own = own[dom[0]] / (dom[2] * 1e-3) / 1e9
    traffic = traffic_src = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
        traffic = tj.get(dom[0])
        traffic_src = {"source": tj.get("_source"), "commit": tj.get("_commit"),
                       "note": "DRAM read+write per launch from the ncu --set full capture at that "
                               "commit (not measured in this run)"}
    except Exception:
        pass
    pf = demag_flops(g, kern)
    fp64 = None
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
            fpk = float(json.load(f)["fp64_tflops"])
        t_yz = (passes[1] + passes[2] + passes[3]) * 1e-3
        fp64 = {"gflop_per_eval": sum(pf) / 1e9, "eval_tflops": sum(pf) / (ms_eval.value * 1e-3) / 1e12,
                "yz_tflops": (pf[1] + pf[2] + pf[3]) / t_yz / 1e12, "peak_tflops": fpk,
                "yz_frac": (pf[1] + pf[2] + pf[3]) / t_yz / 1e12 / fpk,
                "peak_source": "profiles/fp64_peak.json (tools/micro/fp64_peak.cu, DFMA chains)",
                "flops": "SURVEY 8d formula"}
    except Exception:
        pass
    step_bytes = stencil_bytes + 4 * sum(pb)
    step_bytes_own = stencil_bytes + 4 * sum(pb_own)
    # end to end through the public API with host buffers
    e2e = e2e_pageable = None
    if not args.no_e2e:
        pinned = C.c_void_p()
        L.check(L.load().mxb_host_alloc(m.data.nbytes, C.byref(pinned)))
        host = np.ctypeslib.as_array((C.c_double * (3 * N)).from_address(pinned.value)).reshape(m.data.shape)
        host[...] = m.data
        # untimed warm-up of the run_until path (first-call setup of the loop)
        mx.Simulation(mx.SimState(mx.VectorField3(g, host.copy())), rhs, mx.IntegratorSpec("rk4", dt),
                      sample_every=1, energy_in_samples=False).run_until(mx.StopCondition(max_steps=1))
        st = mx.SimState(mx.VectorField3(g, host))
        sim = mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", dt), sample_every=1,
                            energy_in_samples=False)
        sim.CHUNK = 1
        t0 = time.perf_counter()
        sim.run_until(mx.StopCondition(max_steps=args.steps))
        el = time.perf_counter() - t0
        e2e = {"value": N * args.steps / el, "unit": "cell-steps/s",
               "h2d_bytes_per_step": int(24 * N / args.steps),
               "d2h_bytes_per_step": int(24 * N / args.steps + 24),
               "note": "Simulation.run_until from pinned host state; <m> read back every step"}
        del st, sim
        L.load().mxb_host_free(pinned)
        # the reference API's normal input: a plain (pageable) numpy state
        st = mx.SimState(mx.VectorField3(g, m.data.copy()))
        sim = mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", dt), sample_every=1,
                            energy_in_samples=False)
        sim.CHUNK = 1
        t0 = time.perf_counter()
        sim.run_until(mx.StopCondition(max_steps=args.steps))
        el = time.perf_counter() - t0
        e2e_pageable = {"value": N * args.steps / el, "unit": "cell-steps/s",
                        "h2d_bytes_per_step": int(24 * N / args.steps),
                        "d2h_bytes_per_step": int(24 * N / args.steps + 24),
                        "note": "Simulation.run_until from a pageable numpy state; <m> every step"}
        del st, sim
    cpu = None
    if rank == 0 and not args.no_cpu:
        cs, el, cores = cpu_reference(args.cpu_n, 5, 1)
        cpu = {"value": cs, "unit": "cell-steps/s", "cores": cores, "kind": "port",
               "sample": f"synthetic {args.cpu_n}^3 full H_eff, 1 warm-up + 5 timed RK4 steps, oracle "
                         f"numpy/scipy (tensor build excluded)",
               "extrapolated_to_size": extrapolate_cpu(cs, args.cpu_n, args.size)}
    dev = tensor_deviation(mx) if not args.no_dev else None
    cmode = None
    if not args.no_ref_mode:
        cmode = complex_mode(mx, L, C, ctx, g, ts, dt, bptr, args)
    if rank != 0:
        return
    out = {
        "metric": METRIC, "value": value, "unit": "cell-steps/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"synthetic random-m {args.size}^3, full H_eff "
                               "(demag+exchange+DMI+uniaxial anis+Zeeman), RK4",
                   "cells": N, "dt": dt, "l2": "inputs (3.2 GB/field) > L2, no flush",
                   "parallelism": "single GPU"},
        "roofline": {"bound": "hbm", "kernel": dom[0], "achieved": ach, "peak": hbm,
                     "unit": "GB/s", "frac": ach / hbm, "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": which, "bytes": "SURVEY 8d fixed formula",
                     "achieved_impl_bytes": ach_own, "frac_impl_bytes": ach_own / hbm,
                     "frac_vs_8TBs_nominal": ach / 8000.0},
        "step_roofline": {"bytes_per_step": step_bytes,
                          "achieved_GBs": step_bytes / (t_step * 1e-3) / 1e9,
                          "frac": step_bytes / (t_step * 1e-3) / 1e9 / hbm,
                          "bytes_per_step_impl": step_bytes_own,
                          "frac_impl_bytes": step_bytes_own / (t_step * 1e-3) / 1e9 / hbm,
                          "frac_vs_8TBs_nominal": step_bytes / (t_step * 1e-3) / 1e9 / 8000.0},
        "kernels_ms_per_step": share,
        "timing": {"repeats": len(runs), "ms_per_step_runs": runs, "statistic": "median",
                   "clock": "CUDA events on the solver stream"},
        "fp64": fp64,
        "demag_ms_per_eval": ms_eval.value, "cufft_demag_ms_per_eval": ms_cufft.value,
        "tensor_build_s": t_build,
        "tensor": {"build": "GPU Newell tensor (newell.cu) with correctly rounded atan/asinh "
                            "(dd_math.cuh); mirrored octant (symmetric=True), real parity-reduced spectra",
                   "kmode": kern.kmode, "deviation_vs_reference": dev,
                   "deviation_tests": "tests/test_bench_path_parity.py (32/64/128^3) and "
                                      "tests/test_tensor_noise_floor.py (the reference's own "
                                      "cross-host spread)"},
        "reference_tensor_mode": cmode,
        "e2e": e2e, "e2e_pageable": e2e_pageable, "cpu_baseline": cpu, "gpu_launches": int(nl.value),
        "clocks": clk.summary(),
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
