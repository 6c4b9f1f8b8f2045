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


def problem():
    mat = O.make_mat((NX, NY, NZ), CELL, 8e5, A=1.3e-11, Ku=5e4, eK=(0.3, 0.2, 1.0), D=1e-3,
                     alpha=0.1)
    rng = np.random.default_rng(21)
    m0 = O.renormalize(rng.normal(size=(3, NZ, NY, NX)), mat)
    packed = O.packed_tensor(NX, NY, NZ, *CELL)
    return mat, m0, packed


def reference():
    mat, m0, packed = problem()
    terms = O.Terms(exchange=True, anisotropy=True, dmi=True, spectra=O.kernel_spectra(packed),
                    bias=np.array(BIAS))
    return O.run(m0, mat, terms, "rk4", DT, max_steps=NSTEPS, sample_every=1)


def _terms():
    from paper_2602_12242_b200 import _lib as L
    return L.Terms(L.TERM_EXCHANGE | L.TERM_ANISOTROPY | L.TERM_DMI | L.TERM_DEMAG | L.TERM_BIAS,
                   L.GHOST["dmi"], 1, 1)


def _worker(rank, world, port, kind, out):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2602_12242_b200.slab import Comm, SlabPlan, SlabSimulation
    mat, m0, packed = problem()
    plan = SlabPlan(NX, NY, NZ, world, rank)
    z0, nzl = plan.z0, plan.nz_local
    terms = _terms()
    if kind == "numpy":
        from tests.slab_numpy import NumpySlabBackend
        b = NumpySlabBackend(plan, mat, O.kernel_spectra(packed), terms)
    else:
        import ctypes as C

        import paper_2602_12242_b200 as mx
        from paper_2602_12242_b200 import _lib as L
        from paper_2602_12242_b200.slab import CudaSlabBackend
        torch.cuda.set_device(0)
        gl = mx.GridSpec(NX, NY, nzl, *CELL)
        mat_l = mx.MaterialMap(gl, Ms=8e5, A=1.3e-11, Ku=5e4, eK=(0.3, 0.2, 1.0), D=1e-3, alpha=0.1)
        h = C.c_void_p()
        L.check(L.load().mxb_demag_create_slab(C.byref(mx.GridSpec(NX, NY, NZ, *CELL)._c()), 0, world,
                                               rank, C.byref(h)))
        L.check(L.load().mxb_demag_set_packed(h, L.dptr(np.ascontiguousarray(packed))))
        b = CudaSlabBackend(plan, gl, mat_l, h, 0)
    sim = SlabSimulation(plan, b, Comm(), terms, method="rk4", dt=DT, bias=BIAS)
    sim.start(m0[:, z0:z0 + nzl])
    st = sim.run(NSTEPS)
    out[rank] = (sim.state(), st.steps_done, np.array(st.mean[:3]), st.status)
    dist.destroy_process_group()


def _run(kind):
    world = 2
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, free_port(), kind, out), nprocs=world,
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


def test_slab_numpy_gloo_matches_single_domain():
    ref = reference()
    state, steps, mean0, status, mean1 = _run("numpy")
    assert steps == NSTEPS and status == 0
    assert np.max(np.abs(state - ref.m)) <= 1e-12 * 8e5
    assert np.array_equal(mean0, mean1)              # every rank committed the same step
    assert np.max(np.abs(mean0 - np.array([ref.rows[-1][k] for k in ("mx", "my", "mz")]))) <= 1e-12


@pytest.mark.gpu
def test_slab_cuda_two_ranks_match_single_domain():
    ref = reference()
    state, steps, mean0, status, mean1 = _run("cuda")
    assert steps == NSTEPS and status == 0
    assert np.max(np.abs(state - ref.m)) <= 1e-11 * 8e5
    assert np.array_equal(mean0, mean1)
    assert np.max(np.abs(mean0 - np.array([ref.rows[-1][k] for k in ("mx", "my", "mz")]))) <= 1e-11
