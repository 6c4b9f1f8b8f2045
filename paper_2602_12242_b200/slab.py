"""z-slab decomposition of the fused RK4/Euler loop across ranks.

One process per GPU, ``torch.distributed`` for the plumbing (NCCL over
NVLink on GPUs; gloo on CPU for the tests).  Rank r of G owns the z planes
[r*nz/G, (r+1)*nz/G) of every field.  Per RK stage:

  * demag of the stage state: x r2c of the local rows written straight into
    per-destination kx chunks -> all-to-all -> y / fused z*kernel / y inverse
    on this rank's kx chunk -> all-to-all back -> x c2r (csrc/demag.cu,
    ``mxb_demag_x_forward / yz / x_inverse``).  The transpose sits after the
    x pass, where the data is smallest (48*hx*ny*nz/G bytes per rank).
  * stencil halos: the first and last local planes go to the z-neighbours,
    whose planes arrive as ``halo_lo`` / ``halo_hi`` of the fused stage kernel.
  * after the last stage: the per-rank (sum m/Ms, max drift, halt, dead cell)
    partials are all-reduced and every rank commits the same step
    (blow-up / <m> / residual / equilibrium of llg.py:347-371).

The compute backend is swappable: ``CudaSlabBackend`` runs the sm_100a
kernels; ``tests/slab_numpy.py`` provides a numpy backend built on the oracle
so the orchestration below is exercised under gloo on CPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L


@dataclass(frozen=True)
class SlabPlan:
    """Host-side geometry of the decomposition (mirrors DemagPlan::init)."""

    nx: int
    ny: int
    nz: int
    nranks: int
    rank: int

    def __post_init__(self):
        if self.nz % self.nranks:
            raise ValueError(f"nz={self.nz} is not divisible by {self.nranks} ranks")

    @property
    def nz_local(self) -> int:
        return self.nz // self.nranks

    @property
    def z0(self) -> int:
        return self.rank * self.nz_local

    @property
    def hx(self) -> int:
        return (2 * self.nx if self.nx > 1 else 1) // 2 + 1

    @property
    def chunk(self) -> int:
        return self.hx if self.nranks == 1 else -(-self.hx // self.nranks)

    @property
    def chunk_pitch(self) -> int:
        return (self.chunk + 7) // 8 * 8

    @property
    def kx0(self) -> int:
        return self.rank * self.chunk

    @property
    def kx_count(self) -> int:
        return max(0, min(self.chunk, self.hx - self.kx0))

    @property
    def block_elems(self) -> int:
        """complex elements per all-to-all block"""
        return self.nz_local * self.ny * self.chunk_pitch * 3

    def neighbours(self, periodic: bool):
        lo = self.rank - 1
        hi = self.rank + 1
        if periodic:
            return lo % self.nranks, hi % self.nranks
        return (lo if lo >= 0 else None), (hi if hi < self.nranks else None)


class Comm:
    """Collectives of the slab loop over a torch.distributed process group.

    Device tensors go straight to NCCL; with the gloo backend they are staged
    through host memory (tests)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.staged = dist.get_backend(group) != "nccl"

    def _stage(self, *ts):
        if not self.staged:
            return ts, lambda: None
        host = tuple(t.detach().cpu() for t in ts)

        def back():
            for t, h in zip(ts, host):
                t.copy_(h)

        return host, back

    def alltoall(self, out, inp):
        (o, i), back = self._stage(out, inp)
        self.dist.all_to_all_single(o, i, group=self.group)
        back()

    def allreduce(self, t, op: str):
        (h,), back = self._stage(t)
        self.dist.all_reduce(h, op=self.dist.ReduceOp.SUM if op == "sum" else self.dist.ReduceOp.MAX,
                             group=self.group)
        back()

    def halos(self, send_lo, send_hi, recv_lo, recv_hi, lo_rank, hi_rank):
        """send_lo -> lo_rank (it becomes that rank's halo_hi), send_hi -> hi_rank;
        receive the neighbours' boundary planes into recv_lo / recv_hi."""
        ts = [t for t in (send_lo, send_hi, recv_lo, recv_hi)]
        hs, back = self._stage(*ts)
        s_lo, s_hi, r_lo, r_hi = hs
        ops = []
        P2P = self.dist.P2POp
        if lo_rank is not None:
            ops += [P2P(self.dist.isend, s_lo, self._g(lo_rank), self.group),
                    P2P(self.dist.irecv, r_lo, self._g(lo_rank), self.group)]
        if hi_rank is not None:
            ops += [P2P(self.dist.isend, s_hi, self._g(hi_rank), self.group),
                    P2P(self.dist.irecv, r_hi, self._g(hi_rank), self.group)]
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()
        back()

    def _g(self, r):
        return r if self.group is None else self.dist.get_global_rank(self.group, r)


class _CudaArray:
    """__cuda_array_interface__ view of library-owned device memory."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None}


class CudaSlabBackend:
    """One rank's slab on its GPU: fields as torch tensors, kernels from libmagnex_b200."""

    def __init__(self, plan: SlabPlan, grid, mat_local, demag_handle, device: int):
        import torch
        self.torch = torch
        self.plan = plan
        self.dev = torch.device("cuda", device)
        self.mat = mat_local
        self.ctx = mat_local._ctx()
        self.d = demag_handle
        # torch's legacy default stream has handle 0; pass cudaStreamLegacy (0x1)
        # so our kernels are ordered with torch's copies and collectives
        self.stream = torch.cuda.current_stream(self.dev).cuda_stream or 1
        lib = L.load()
        L.check(lib.mxb_ctx_set_stream(self.ctx.h, C.c_void_p(self.stream)))
        shape = (3, plan.nz_local, plan.ny, plan.nx)
        self.fields = {k: torch.zeros(shape, dtype=torch.float64, device=self.dev)
                       for k in ("Y0", "Y1", "P", "K1", "S", "HD")}
        hshape = (3, plan.ny, plan.nx)
        self.halo = {k: torch.zeros(hshape, dtype=torch.float64, device=self.dev)
                     for k in ("send_lo", "send_hi", "lo", "hi")}
        self.red = torch.zeros(8, dtype=torch.float64, device=self.dev)
        self.mhalo = None   # neighbour planes of (Ms, A): set by material_halos
        if self.d is not None:
            L.check(lib.mxb_demag_set_stream(self.d, C.c_void_p(self.stream)))
            s, r = C.c_void_p(), C.c_void_p()
            L.check(lib.mxb_demag_slab_buffers(self.d, C.byref(s), C.byref(r)))
            blk = C.c_int64()
            L.check(lib.mxb_demag_slab_block(self.d, C.byref(blk)))
            # row-major kx chunks (plan.block_elems) or, with the plane pipeline,
            # plane-major chunks of whole kx planes
            n = 2 * plan.nranks * int(blk.value)
            self.send = torch.as_tensor(_CudaArray(s.value, n), device=self.dev)
            self.recv = torch.as_tensor(_CudaArray(r.value, n), device=self.dev)

    # -- data movement -----------------------------------------------------------
    def upload(self, name, host):
        self.fields[name].copy_(self.torch.from_numpy(np.ascontiguousarray(host)))

    def download(self, name):
        return self.fields[name].cpu().numpy()

    def boundary_planes(self, name):
        # both boundary planes of the three components in one kernel (mxb_pack_halo_planes)
        L.check(self.ctx.call("mxb_pack_halo_planes", C.c_void_p(self.fields[name].data_ptr()),
                              C.c_void_p(self.halo["send_lo"].data_ptr()),
                              C.c_void_p(self.halo["send_hi"].data_ptr())), "pack_halo")
        return self.halo["send_lo"], self.halo["send_hi"], self.halo["lo"], self.halo["hi"]

    def material_halos(self, comm, lo_rank, hi_rank):
        """Swap the boundary planes of Ms and A with the z-neighbours once, so
        the stage kernel sees the neighbours' material across the slab faces
        (validity and the harmonic exchange coefficient, fields.py:59-92)."""
        if lo_rank is None and hi_rank is None:
            return
        mat, p = self.mat, self.plan
        shape = (p.nz_local, p.ny, p.nx)
        Ms = np.broadcast_to(mat.Ms, shape)
        A = np.broadcast_to(mat.A, shape)
        send_lo = self.new_tensor(np.stack([Ms[0], A[0]]))
        send_hi = self.new_tensor(np.stack([Ms[-1], A[-1]]))
        recv_lo = self.torch.zeros_like(send_lo)
        recv_hi = self.torch.zeros_like(send_hi)
        comm.halos(send_lo, send_hi, recv_lo, recv_hi, lo_rank, hi_rank)
        if mat._Ms_u is not None and mat._A_u is not None:
            # uniform local material: the uniform kernels take the neighbours'
            # material to be the local one -- check that it is
            for r, rk in ((recv_lo, lo_rank), (recv_hi, hi_rank)):
                if rk is None:
                    continue
                h = r.cpu().numpy()
                if np.any(h[0] != mat._Ms_u) or np.any(h[1] != mat._A_u):
                    raise ValueError("the material changes across a slab boundary but is uniform on this "
                                     "rank; pass it per cell (a non-uniform MaterialMap) on every rank")
            return
        self.mhalo = (recv_lo, recv_hi)

    # -- demag ----------------------------------------------------------------------
    def demag_x_forward(self, src):
        L.check(L.load().mxb_demag_x_forward(self.d, C.c_void_p(self.fields[src].data_ptr())))

    def demag_yz(self):
        L.check(L.load().mxb_demag_yz(self.d))

    def demag_x_inverse(self, dst):
        L.check(L.load().mxb_demag_x_inverse(self.d, C.c_void_p(self.fields[dst].data_ptr())))

    # -- stencil stage ----------------------------------------------------------------
    def stage(self, mode, terms: L.Terms, *, ys, y, out, hd=None, k1=None, s=None, k1_out=None,
              halo_lo=False, halo_hi=False, bias=(0.0, 0.0, 0.0), c=0.0, dt6=0.0, renorm=True):
        f = self.fields
        io = L.StageIO()
        ptr = lambda name: C.c_void_p(f[name].data_ptr()) if name else None  # noqa: E731
        io.ys, io.y, io.out = ptr(ys), ptr(y), ptr(out)
        io.hd, io.k1, io.s, io.k1_out = ptr(hd), ptr(k1), ptr(s), ptr(k1_out)
        io.halo_lo = C.c_void_p(self.halo["lo"].data_ptr()) if halo_lo else None
        io.halo_hi = C.c_void_p(self.halo["hi"].data_ptr()) if halo_hi else None
        if self.mhalo is not None:
            lo, hi = self.mhalo
            plane = lo.shape[1] * lo.shape[2] * 8
            if halo_lo:
                io.hms_lo, io.hA_lo = C.c_void_p(lo.data_ptr()), C.c_void_p(lo.data_ptr() + plane)
            if halo_hi:
                io.hms_hi, io.hA_hi = C.c_void_p(hi.data_ptr()), C.c_void_p(hi.data_ptr() + plane)
        io.bias = (C.c_double * 3)(*bias)
        io.c, io.dt6, io.renorm = c, dt6, 1 if renorm else 0
        L.check(self.ctx.call("mxb_stage_dev", mode, C.byref(terms), C.byref(io)), "stage")

    def partials(self):
        L.check(self.ctx.call("mxb_step_partials_dev", C.c_void_p(self.red.data_ptr())))
        return self.red

    def commit(self, totals):
        L.check(self.ctx.call("mxb_step_commit_dev", C.c_void_p(totals.data_ptr())))

    def ctl_reset(self, prev_mean, n_magnetic, eq_tol):
        p = np.ascontiguousarray(prev_mean, dtype=np.float64)
        L.check(self.ctx.call("mxb_ctl_reset", L.dptr(p), int(n_magnetic), float(eq_tol)))

    def ctl_get(self):
        st = L.RunStats()
        L.check(self.ctx.call("mxb_ctl_get", C.byref(st)))
        return st

    def local_mean_sums(self, name):
        """sum of m/Ms over local magnetic cells (for the initial <m>)"""
        m = self.download(name)
        mask = self.mat.mask
        with np.errstate(invalid="ignore", divide="ignore"):
            q = m / np.where(mask, self.mat.Ms, 1.0)
        return np.array([q[c][mask].sum() for c in range(3)]), int(np.count_nonzero(mask))

    def new_tensor(self, host):
        return self.torch.as_tensor(np.asarray(host, dtype=np.float64), device=self.dev)


RK4_STAGES = (  # (mode, ys, out, coefficient, uses k1/s)
    (2, "Y", "P", 0.5),
    (3, "P", "YN", 0.5),
    (4, "YN", "P", 1.0),
    (5, "P", "YN", None),
)


class SlabSimulation:
    """Fixed-step RK4/Euler loop on a z-slab (the multi-rank Simulation.run_until core)."""

    def __init__(self, plan: SlabPlan, backend, comm: Comm, terms: L.Terms, *, method="rk4",
                 dt: float, bias=None, periodic_z=False, use_demag=True, renorm_each_stage=True,
                 check_every: int = 16):
        if method not in ("rk4", "euler"):
            raise ValueError(f"unknown method {method!r}")
        self.plan, self.b, self.comm, self.terms = plan, backend, comm, terms
        self.method, self.dt = method, float(dt)
        self.bias = bias
        self.use_demag = use_demag
        self.renorm = renorm_each_stage
        self.lo_rank, self.hi_rank = plan.neighbours(periodic_z)
        self.cur = "Y0"
        self.t0 = 0.0
        self.step = 0
        # the step commit runs on the device (every rank applies the same
        # all-reduced totals; after a halt the stage kernels are no-ops), so the
        # host reads the control block only every check_every steps
        self.check_every = max(1, int(check_every))

    def _bias_at(self, t):
        if self.bias is None:
            return (0.0, 0.0, 0.0)
        v = self.bias(t) if callable(self.bias) else self.bias
        return tuple(float(x) for x in np.asarray(v, dtype=np.float64))

    def _demag(self, src):
        b = self.b
        b.demag_x_forward(src)
        if self.comm.size > 1:
            self.comm.alltoall(b.recv, b.send)
        b.demag_yz()
        if self.comm.size > 1:
            self.comm.alltoall(b.send, b.recv)
        b.demag_x_inverse("HD")

    def _halos(self, src):
        if self.comm.size == 1 and self.lo_rank is None:
            return False, False
        send_lo, send_hi, recv_lo, recv_hi = self.b.boundary_planes(src)
        self.comm.halos(send_lo, send_hi, recv_lo, recv_hi, self.lo_rank, self.hi_rank)
        return self.lo_rank is not None, self.hi_rank is not None

    def start(self, m_local, eq_tol=None, t0: float = 0.0):
        b = self.b
        self.t0, self.step = float(t0), 0
        b.upload("Y0", m_local)
        self.cur = "Y0"
        sums, nmag = b.local_mean_sums("Y0")
        tot = b.new_tensor(np.concatenate([sums, [nmag]]))
        self.comm.allreduce(tot, "sum")
        tot = tot.cpu().numpy()
        self.n_magnetic = int(round(tot[3]))
        self.mean0 = tot[:3] / self.n_magnetic
        b.ctl_reset(self.mean0, self.n_magnetic, -1.0 if eq_tol is None else eq_tol)
        if hasattr(b, "material_halos"):
            b.material_halos(self.comm, self.lo_rank, self.hi_rank)

    def run(self, nsteps: int):
        """Advance up to nsteps; stops early on blow-up, a dead cell or equilibrium.
        Time is t0 + k*dt (llg.py:357); stage times t, t+dt/2, t+dt/2, t+dt."""
        b, dt = self.b, self.dt
        nxt = {"Y0": "Y1", "Y1": "Y0"}
        if self.method == "euler":
            stages, offs = ((6, "Y", "YN", 1.0),), (0.0,)
        else:
            stages, offs = RK4_STAGES, (0.0, 0.5 * dt, 0.5 * dt, dt)
        st = b.ctl_get()
        done0 = int(st.steps_done)
        cur0, step0 = self.cur, self.step
        for i in range(nsteps):
            # issued as if every step commits; corrected from steps_done at each check
            y, yn = self.cur, nxt[self.cur]
            tb = self.t0 + self.step * dt
            for (mode, ys, out, c), off in zip(stages, offs):
                ys = y if ys == "Y" else (yn if ys == "YN" else ys)
                out = yn if out == "YN" else out
                if self.use_demag:
                    self._demag(ys)
                lo, hi = self._halos(ys)
                b.stage(mode, self.terms, ys=ys, y=y, out=out, hd="HD" if self.use_demag else None,
                        k1="K1", s="S", k1_out="K1", halo_lo=lo, halo_hi=hi,
                        bias=self._bias_at(tb if off == 0.0 else tb + off),
                        c=(c or 0.0) * dt, dt6=dt / 6.0,
                        renorm=self.renorm if mode in (2, 3, 4) else True)
            p = b.partials()
            s, mx = p[:4].clone(), p[4:].clone()
            self.comm.allreduce(s, "sum")
            self.comm.allreduce(mx, "max")
            b.commit(b.torch.cat([s, mx]))
            self.cur = yn
            self.step += 1
            if (i + 1) % self.check_every == 0 or i + 1 == nsteps:
                st = b.ctl_get()
                done = int(st.steps_done) - done0
                self.step = step0 + done
                self.cur = cur0 if done % 2 == 0 else nxt[cur0]
                if st.status != 0:
                    break
        return st

    def state(self):
        return self.b.download(self.cur)
