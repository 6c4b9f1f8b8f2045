"""Debug driver for the CUDA slab path: run under torchrun with gloo, e.g.
torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/debug_slab.py
Prints per-rank errors of the distributed demag and of one stencil stage."""
import ctypes as C
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2602_12242_b200 as mx  # noqa: E402
from oracle import magnex_oracle as O  # noqa: E402
from paper_2602_12242_b200 import _lib as L  # noqa: E402
from paper_2602_12242_b200.slab import Comm, CudaSlabBackend, SlabPlan  # noqa: E402
from tests.test_slab import BIAS, CELL, NX, NY, NZ, _terms, problem  # noqa: E402

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
mat, m0, packed = problem()
plan = SlabPlan(NX, NY, NZ, world, rank)
z0, nzl = plan.z0, plan.nz_local
gl = mx.GridSpec(NX, NY, nzl, *CELL)
mat_l = mx.MaterialMap(gl, Ms=8e5, A=1.3e-11, Ku=5e4, eK=(0.3, 0.2, 1.0), D=1e-3, alpha=0.1)
h = C.c_void_p()
L.check(L.load().mxb_demag_create_slab(C.byref(mx.GridSpec(NX, NY, NZ, *CELL)._c()), 0, world, rank,
                                       C.byref(h)))
L.check(L.load().mxb_demag_set_packed(h, L.dptr(np.ascontiguousarray(packed))))
info = (C.c_int64 * 8)()
L.load().mxb_demag_slab_info(h, info)
print(rank, "slab info", list(info), "plan", plan.nz_local, plan.z0, plan.chunk, plan.chunk_pitch,
      plan.kx0, plan.kx_count, plan.block_elems, flush=True)
b = CudaSlabBackend(plan, gl, mat_l, h, 0)
comm = Comm()
b.upload("Y0", m0[:, z0:z0 + nzl])
b.demag_x_forward("Y0")
if world > 1:
    comm.alltoall(b.recv, b.send)
b.demag_yz()
if world > 1:
    comm.alltoall(b.send, b.recv)
b.demag_x_inverse("HD")
hd = b.download("HD")
ref = O.demag_field(O.kernel_spectra(packed), m0)[:, z0:z0 + nzl]
print(rank, "demag err", np.max(np.abs(hd - ref)) / np.max(np.abs(ref)), flush=True)
# one H_eff stage with halos
lo_r, hi_r = plan.neighbours(False)
sl, sh, rl, rh = b.boundary_planes("Y0")
comm.halos(sl, sh, rl, rh, lo_r, hi_r)
terms = _terms()
b.stage(0, terms, ys="Y0", y="Y0", out="P", hd="HD", halo_lo=lo_r is not None,
        halo_hi=hi_r is not None, bias=BIAS)
heff = b.download("P")
to = O.Terms(exchange=True, anisotropy=True, dmi=True, spectra=O.kernel_spectra(packed),
             bias=np.array(BIAS))
href = O.h_eff(0.0, m0, mat, to)[:, z0:z0 + nzl]
err = np.abs(heff - href)
print(rank, "heff err", err.max() / np.abs(href).max(), "worst plane", np.unravel_index(err.argmax(), err.shape),
      flush=True)
dist.destroy_process_group()
