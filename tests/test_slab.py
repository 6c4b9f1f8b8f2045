"""z-slab decomposition: world-size-2 torch.distributed runs vs the single
domain oracle.  The CPU test drives SlabSimulation with the numpy backend
under gloo; the GPU test drives it with the CUDA kernels (two ranks sharing
cuda:0, gloo collectives staged through host memory -- no kernel ever waits
on another rank)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import magnex_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

NX, NY, NZ = 16, 8, 8
# grids of the plane-pipeline slab cases (ny == nz; MXB_PIPE=1 forces the pipeline):
# radix-16 core (L = 32), warp pair core (L = 512), warp core (L = 1024, the bench's)
# pipe512 / pipe1024 run the reference's tensor (complex-spectra pipeline, kernel
# mode 5); pipe1024sym the mirrored GPU build (kernel mode 3, the bench's mode),
# checked against the single-domain oracle on the spectra of the same build
PIPE_DIMS = {"pipe512": (8, 256, 256), "pipe1024": (8, 512, 512), "pipe1024sym": (8, 512, 512),
             # long y lines (py = 2048, the film's path: k_yrow + the fused z pass), mirrored build
             "longysym": (8, 1024, 8)}
CELL = (2e-9, 2.5e-9, 3e-9)
DT = 2e-14
NSTEPS = 3
BIAS = (1e4, -2e3, 5e3)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def dims_of(case):
    return PIPE_DIMS.get(case, (NX, NY, NZ))


def _disk_ms():
    y, x = np.mgrid[0:NY, 0:NX]
    inside = ((x - (NX - 1) / 2) / (NX / 2)) ** 2 + ((y - (NY - 1) / 2) / (NY / 2)) ** 2 <= 1.0
    return np.broadcast_to(np.where(inside, 8e5, 0.0), (NZ, NY, NX)).copy()


def _mat_kw(case):
    """uniform: the round-1 problem; disk: per-cell Ms (vacuum outside an
    elliptic disk), A varying along z (so the slab faces see a different
    neighbour A), plus cubic anisotropy and bulk DMI."""
    kw = dict(A=1.3e-11, Ku=5e4, eK=(0.3, 0.2, 1.0), D=1e-3, alpha=0.1)
    if case == "disk":
        kw["A"] = 1.3e-11 * (1.0 + 0.1 * np.arange(NZ))[:, None, None] * np.ones((NZ, NY, NX))
        kw.update(Kc1=3e4, c1=(1.0, 1.0, 0.0), c2=(-1.0, 1.0, 0.5), Db=1.2e-3)
        return _disk_ms(), kw
    return 8e5, kw


def problem(case="uniform"):
    nx, ny, nz = dims_of(case)
    ms, kw = _mat_kw(case)
    mat = O.make_mat((nx, ny, nz), CELL, ms, **kw)
    rng = np.random.default_rng(21)
    m0 = O.renormalize(rng.normal(size=(3, nz, ny, nx)), mat)
    packed = O.packed_tensor(nx, ny, nz, *CELL)
    return mat, m0, packed


def _sym_spectra(case):
    import paper_2602_12242_b200 as mx
    return mx.DemagKernel.build(mx.GridSpec(*dims_of(case), *CELL), symmetric=True).spectra


def reference(case="uniform"):
    mat, m0, packed = problem(case)
    extra = case == "disk"
    spectra = _sym_spectra(case) if case.endswith("sym") else O.kernel_spectra(packed)
    terms = O.Terms(exchange=True, anisotropy=True, dmi=True, spectra=spectra,
                    bias=np.array(BIAS), cubic=extra, bulk_dmi=extra)
    return O.run(m0, mat, terms, "rk4", DT, max_steps=NSTEPS, sample_every=1)


def reference_state(case):
    """the single-domain result (cached per case: the large pipeline grids take
    seconds per oracle evaluation)"""
    if case not in _REF:
        _REF[case] = reference(case)
    return _REF[case]


_REF = {}


def _terms(case="uniform"):
    from paper_2602_12242_b200 import _lib as L
    mask = L.TERM_EXCHANGE | L.TERM_ANISOTROPY | L.TERM_DMI | L.TERM_DEMAG | L.TERM_BIAS
    if case == "disk":
        mask |= L.TERM_CUBIC | L.TERM_BULK_DMI
    return L.Terms(mask, L.GHOST["dmi"], 1, 1)


def _worker(rank, world, port, kind, out, case="uniform", check_every=16):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if case in PIPE_DIMS and not case.startswith("longy"):
        os.environ["MXB_PIPE"] = "1"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2602_12242_b200.slab import Comm, SlabPlan, SlabSimulation
    mat, m0, packed = problem(case)
    NX_, NY_, NZ_ = dims_of(case)
    plan = SlabPlan(NX_, NY_, NZ_, world, rank)
    z0, nzl = plan.z0, plan.nz_local
    terms = _terms(case)
    if kind == "numpy":
        from tests.slab_numpy import NumpySlabBackend
        b = NumpySlabBackend(plan, mat, O.kernel_spectra(packed), terms)
    else:
        import ctypes as C

        import paper_2602_12242_b200 as mx
        from paper_2602_12242_b200 import _lib as L
        from paper_2602_12242_b200.slab import CudaSlabBackend
        torch.cuda.set_device(0)
        gl = mx.GridSpec(NX_, NY_, nzl, *CELL)
        ms, kw = _mat_kw(case)
        sl = (lambda a: a[z0:z0 + nzl] if np.ndim(a) == 3 else a)  # noqa: E731
        kw = {k: sl(v) for k, v in kw.items()}
        mat_l = mx.MaterialMap(gl, Ms=sl(ms), **kw)
        h = C.c_void_p()
        L.check(L.load().mxb_demag_create_slab(C.byref(mx.GridSpec(NX_, NY_, NZ_, *CELL)._c()), 0, world,
                                               rank, C.byref(h)))
        if case.endswith("sym"):
            L.check(L.load().mxb_demag_build(h, 1))
        else:
            L.check(L.load().mxb_demag_set_packed(h, L.dptr(np.ascontiguousarray(packed))))
        km = C.c_int()
        L.check(L.load().mxb_demag_kmode(h, C.byref(km)))
        if case.startswith("longy"):
            assert km.value == 4, km.value       # long-y path on the rank's kx chunk
        elif case in PIPE_DIMS:
            # plane pipeline: mirrored build -> real quarter (3), reference tensor -> complex (5)
            assert km.value == (3 if case.endswith("sym") else 5), km.value
        b = CudaSlabBackend(plan, gl, mat_l, h, 0)
    sim = SlabSimulation(plan, b, Comm(), terms, method="rk4", dt=DT, bias=BIAS, check_every=check_every)
    sim.start(m0[:, z0:z0 + nzl])
    st = sim.run(NSTEPS)
    out[rank] = (sim.state(), st.steps_done, np.array(st.mean[:3]), st.status)
    dist.destroy_process_group()


def _run(kind, case="uniform", check_every=16, world=2):
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, free_port(), kind, out, case, check_every), nprocs=world,
                       start_method="spawn", join=True)
    state = np.concatenate([out[r][0] for r in range(world)], axis=1)
    return state, out[0][1], out[0][2], out[0][3], out[1][2]


def test_slab_plan_chunks_cover_the_spectrum():
    from paper_2602_12242_b200.slab import SlabPlan
    for nx, g in ((512, 8), (16, 2), (100, 4), (6, 3)):
        covered = []
        for r in range(g):
            p = SlabPlan(nx, 4, 2 * g, g, r)
            covered += list(range(p.kx0, p.kx0 + p.kx_count))
            assert p.chunk_pitch % 8 == 0 and p.chunk_pitch >= p.chunk
        assert covered == list(range(nx + 1))
    with pytest.raises(ValueError):
        SlabPlan(8, 8, 6, 4, 0)


@pytest.mark.parametrize("case,check_every,world", [("uniform", 16, 2), ("uniform", 1, 2), ("disk", 2, 2),
                                                    ("disk", 16, 4)])
def test_slab_numpy_gloo_matches_single_domain(case, check_every, world):
    ref = reference(case)
    state, steps, mean0, status, mean1 = _run("numpy", case, check_every, world)
    assert steps == NSTEPS and status == 0
    assert np.max(np.abs(state - ref.m)) <= 1e-12 * 8e5
    assert np.array_equal(mean0, mean1)              # every rank committed the same step
    assert np.max(np.abs(mean0 - np.array([ref.rows[-1][k] for k in ("mx", "my", "mz")]))) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("case,world", [("uniform", 2), ("disk", 2), ("disk", 4), ("pipe512", 2), ("pipe512", 4),
                                        ("pipe1024", 2), ("pipe1024sym", 2), ("pipe1024sym", 4),
                                        ("longysym", 2), ("longysym", 4)])
def test_slab_cuda_ranks_match_single_domain(case, world):
    """disk: per-cell Ms and A across the slab faces (the neighbours' material
    planes are swapped once at start), cubic anisotropy and bulk DMI.
    pipe*: the y/z plane pipeline on each rank's kx chunk, reading the
    all-to-all receive blocks in place (plane-major chunks)."""
    ref = reference_state(case)
    state, steps, mean0, status, mean1 = _run("cuda", case, world=world)
    assert steps == NSTEPS and status == 0
    assert np.max(np.abs(state - ref.m)) <= 1e-11 * 8e5
    assert np.array_equal(mean0, mean1)
    assert np.max(np.abs(mean0 - np.array([ref.rows[-1][k] for k in ("mx", "my", "mz")]))) <= 1e-11
