"""LLG dynamics: torque, partitioned RHS and the fixed-step driver (reference: llg.py).

``Simulation.run_until`` keeps the state resident on the GPU and advances it
with the fused stage kernels (csrc/stencil.cu) plus the FFT demag
(csrc/demag.cu), in chunks between sample points.  Blow-up, dead cells and
the equilibrium stop are detected on the device at the exact step
(llg.py:346-371).  The host only evaluates time-dependent bias callables at
the stage times, builds sample rows and talks to the caller.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from . import io as mio
from .demag import DemagKernel
from .fields import (AnisotropyOperator, BulkDmiOperator, CubicAnisotropyOperator, DmiOperator,
                     EnergyBreakdown, ExchangeOperator, _StencilPlan)
from .grid import MaterialMap, RenormalizeError, VectorField3, _raise_dead, mean_normalized, renormalize
from .integrators import (_PHASE_WIDTH, KW3_C, euler_step, fast_evals_per_step, mri_kw3_step, rk4_step,
                          substeps_per_phase)

__all__ = ["SLOW_EXPLICIT", "FAST", "SLOW_IMPLICIT", "TERMS", "llg_rhs", "PartitionedRHS",
           "IntegratorSpec", "StopCondition", "SimState", "Trajectory", "Simulation",
           "IntegrationBlowup", "BLOWUP_DRIFT"]

TERMS = ("exchange", "anisotropy", "dmi", "demag", "bias")
EXTRA_TERMS = ("cubic", "bulk_dmi")
SLOW_EXPLICIT = "slow-explicit"
FAST = "fast"
SLOW_IMPLICIT = "slow-implicit"
DEFAULT_PARTITION = {"exchange": FAST, "anisotropy": SLOW_EXPLICIT, "dmi": SLOW_EXPLICIT,
                     "demag": SLOW_EXPLICIT, "bias": SLOW_EXPLICIT, "cubic": SLOW_EXPLICIT,
                     "bulk_dmi": SLOW_EXPLICIT}
BLOWUP_DRIFT = 0.10
_BIT = {"exchange": L.TERM_EXCHANGE, "anisotropy": L.TERM_ANISOTROPY, "dmi": L.TERM_DMI,
        "demag": L.TERM_DEMAG, "bias": L.TERM_BIAS, "cubic": L.TERM_CUBIC,
        "bulk_dmi": L.TERM_BULK_DMI}
# device accumulation order (csrc/stencil.cu heff_cell) == reference order
_ORDER = ("exchange", "anisotropy", "cubic", "dmi", "bulk_dmi", "demag", "bias")


class IntegrationBlowup(RuntimeError):
    """llg.py:54-61"""

    def __init__(self, step: int, t: float, drift: float):
        super().__init__(
            f"integration blew up at step {step} (t = {t:.6e} s): "
            f"pre-renormalization |M| drift {drift:.3g} exceeds {BLOWUP_DRIFT:g}")
        self.step = step
        self.t = t
        self.drift = drift


def _field_args(mat, mdata):
    m = np.ascontiguousarray(mdata, dtype=np.float64)
    if m.shape != (3,) + mat.grid.shape:
        raise ValueError(f"field shape {m.shape} does not match grid {(3,) + mat.grid.shape}")
    return m


def llg_rhs(m: VectorField3, h_eff: VectorField3, mat: MaterialMap, precession: bool = True,
            damping: bool = True) -> VectorField3:
    """dM/dt of the damped precession law on the GPU (llg.py:64-81)."""
    md = _field_args(mat, m.data)
    hd = _field_args(mat, h_eff.data)
    out = np.empty_like(md)
    L.check(mat._ctx().call("mxb_llg_rhs", int(precession), int(damping), L.dptr(md), L.dptr(hd),
                            L.dptr(out)), "llg_rhs")
    return VectorField3(m.grid, out)


class PartitionedRHS:
    """Effective-field assembly with slow/fast partitions and counters (llg.py:84-203).

    ``demag`` is a :class:`DemagKernel` (device FFT path), any object with
    ``field(mdata)`` or a bare callable (a plugin backend evaluated on its own
    terms, e.g. a surrogate).  ``bias`` is a 3-vector, a (3,nz,ny,nx) field,
    or a callable of t returning either.  ``cubic``/``bulk_dmi`` switch on the
    unpinned extension terms.
    """

    def __init__(self, mat: MaterialMap, *, exchange: bool = True, anisotropy: bool = False,
                 dmi: bool = False, demag=None, bias=None, partition: dict | None = None,
                 precession: bool = True, damping: bool = True, ghost_mode: str | None = None,
                 cubic: bool = False, bulk_dmi: bool = False):
        self.mat = mat
        self.precession = precession
        self.damping = damping
        if ghost_mode is None:
            ghost_mode = "dmi" if dmi else "neumann"
        self.ghost_mode = ghost_mode
        self.plan = _StencilPlan(mat, ghost_mode)
        self._ops = {}
        if exchange:
            self._ops["exchange"] = ExchangeOperator(mat, plan=self.plan)
        if anisotropy:
            self._ops["anisotropy"] = AnisotropyOperator(mat)
        if cubic:
            self._ops["cubic"] = CubicAnisotropyOperator(mat)
        if dmi:
            self._ops["dmi"] = DmiOperator(mat, plan=self.plan)
        if bulk_dmi:
            self._ops["bulk_dmi"] = BulkDmiOperator(mat)
        self._demag_dev = None
        self._demag_fn = None
        if demag is not None:
            dk = demag._device_kernel() if hasattr(demag, "_device_kernel") else None
            if isinstance(demag, DemagKernel):
                self._demag_dev = demag
                fn = demag.field
            elif dk is not None:
                # a plugin with a device evaluation (the FNO surrogate): evaluated
                # inside the fused device step like the FFT kernel
                self._demag_dev = dk
                fn = demag.field
            else:
                fn = demag.field if hasattr(demag, "field") else demag
                self._demag_fn = fn
            self._ops["demag"] = lambda mdata, _f=fn: _f(mdata)
        if bias is not None:
            self.set_bias(bias)
        else:
            self._bias = None
        self.partition = dict(DEFAULT_PARTITION)
        for term, part in (partition or {}).items():
            if term not in TERMS and term not in EXTRA_TERMS:
                raise ValueError(f"unknown field term {term!r}")
            if part == SLOW_IMPLICIT:
                raise ValueError("the slow-implicit partition is reserved and has no integrator")
            if part not in (SLOW_EXPLICIT, FAST):
                raise ValueError(f"unknown partition {part!r} for term {term!r}")
            self.partition[term] = part
        self.counters = {term: 0 for term in self.enabled_terms()}

    def set_bias(self, bias) -> None:
        self._bias = bias if callable(bias) else np.asarray(bias, dtype=np.float64)
        if hasattr(self, "counters") and "bias" not in self.counters:
            self.counters["bias"] = 0

    def enabled_terms(self):
        terms = list(self._ops)
        if getattr(self, "_bias", None) is not None:
            terms.append("bias")
        return tuple(terms)

    def terms_in(self, part: str):
        return tuple(t for t in self.enabled_terms() if self.partition[t] == part)

    def bias_at(self, t: float):
        if self._bias is None:
            return None
        b = self._bias(t) if callable(self._bias) else self._bias
        return np.asarray(b, dtype=np.float64)

    # ---- device evaluation -------------------------------------------------
    def _terms_struct(self, terms) -> L.Terms:
        mask = 0
        for t in terms:
            mask |= _BIT[t]
        return L.Terms(mask, L.GHOST[self.ghost_mode], int(bool(self.precession)),
                       int(bool(self.damping)))

    def _bias_struct(self, terms, t, mdata, keep):
        b = L.Bias()
        if "bias" in terms:
            v = self.bias_at(t)
            if v.shape == (3,):
                b.vec = (C.c_double * 3)(*v)
            else:
                f = np.ascontiguousarray(np.broadcast_to(v, (3,) + self.mat.grid.shape),
                                         dtype=np.float64)
                keep.append(f)
                b.field = L.dptr(f)
        if "demag" in terms and self._demag_fn is not None:
            hd = np.ascontiguousarray(self._demag_fn(mdata), dtype=np.float64)
            keep.append(hd)
            b.demag_field = L.dptr(hd)
        return b

    def _eval(self, fn, terms, t, mdata, count):
        m = _field_args(self.mat, mdata)
        keep = []
        ts = self._terms_struct(terms)
        b = self._bias_struct(terms, t, m, keep)
        out = np.empty_like(m)
        d = self._demag_dev._d.h if (self._demag_dev is not None and "demag" in terms) else None
        L.check(self.mat._ctx().call(fn, d, C.byref(ts), C.byref(b), L.dptr(m), L.dptr(out)), fn)
        if count:
            for term in terms:
                self.counters[term] += 1
        return out

    def _add_term(self, term, t, mdata, h, count):
        h += self._eval("mxb_heff", (term,), t, mdata, count)

    def field_of(self, terms, t: float, mdata: np.ndarray, count: bool = True) -> np.ndarray:
        terms = tuple(x for x in _ORDER if x in terms)
        if not terms:
            return np.zeros_like(np.asarray(mdata, dtype=np.float64))
        return self._eval("mxb_heff", terms, t, mdata, count)

    def _rhs(self, terms, t, mdata):
        terms = tuple(x for x in _ORDER if x in terms)
        return self._eval("mxb_rhs_total", terms, t, mdata, True)

    def rhs_total(self, t: float, mdata: np.ndarray) -> np.ndarray:
        return self._rhs(self.enabled_terms(), t, mdata)

    def rhs_slow(self, t: float, mdata: np.ndarray) -> np.ndarray:
        return self._rhs(self.terms_in(SLOW_EXPLICIT), t, mdata)

    def rhs_fast(self, t: float, mdata: np.ndarray) -> np.ndarray:
        return self._rhs(self.terms_in(FAST), t, mdata)

    def h_total_quiet(self, t: float, mdata: np.ndarray) -> np.ndarray:
        return self.field_of(self.enabled_terms(), t, mdata, count=False)

    def demag_quiet(self, mdata: np.ndarray):
        if "demag" not in self._ops:
            return None
        return self._ops["demag"](mdata)

    def energies(self, t: float, m: VectorField3) -> EnergyBreakdown:
        out = np.zeros(4)
        keep = []
        terms = tuple(x for x in ("demag", "bias") if x in self.enabled_terms())
        ts = self._terms_struct(terms)
        md = _field_args(self.mat, m.data)
        b = self._bias_struct(terms, t, md, keep)
        d = self._demag_dev._d.h if (self._demag_dev is not None and "demag" in terms) else None
        L.check(self.mat._ctx().call("mxb_energies", d, C.byref(ts), C.byref(b), L.dptr(md),
                                     L.dptr(out)), "energies")
        return EnergyBreakdown(*(float(v) for v in out))

    # the device stepping loop can run this RHS without host round trips
    def _device_ok(self) -> bool:
        return self._demag_fn is None


@dataclass
class IntegratorSpec:
    """llg.py:206-222"""

    method: str
    dt: float
    theta: float = 0.1
    renorm_each_stage: bool = True

    def __post_init__(self):
        if self.method not in ("euler", "rk4", "mri-kw3"):
            raise ValueError(f"unknown method {self.method!r}")
        if not self.dt > 0:
            raise ValueError(f"dt must be positive, got {self.dt}")
        if not 0.0 < self.theta <= 1.0:
            raise ValueError(f"theta must be in (0, 1], got {self.theta}")


@dataclass
class StopCondition:
    """llg.py:225-237"""

    max_time: float | None = None
    max_steps: int | None = None
    equilibrium_tol: float | None = None

    def __post_init__(self):
        if self.max_time is None and self.max_steps is None:
            raise ValueError("need max_time or max_steps as a hard cap")


@dataclass
class SimState:
    m: VectorField3
    t: float = 0.0
    step: int = 0


@dataclass
class Trajectory:
    samples: list = field(default_factory=list)
    stop_reason: str = ""
    counters: dict = field(default_factory=dict)
    wall_s: float = 0.0
    final_residual: float = float("nan")

    def column(self, name: str) -> np.ndarray:
        return np.array([row[name] for row in self.samples])

    def write_csv(self, path) -> None:
        mio.write_timeseries_csv(path, self.samples)


def _zero_range(buf, offset: int, nbytes: int) -> None:
    C.memset(buf.ctypes.data + offset, 0, nbytes)


def _prefault(shape, nthreads: int = 8):
    """A fresh float64 array whose pages are being written by `nthreads` host
    threads (ctypes.memset releases the GIL); join the threads before use."""
    buf = np.empty(shape)
    n = buf.nbytes
    step = ((n + nthreads - 1) // nthreads + 4095) // 4096 * 4096
    threads = []
    for o in range(0, n, step):
        # the thread holds `buf` itself, so an abandoned run cannot free it under the memset
        th = threading.Thread(target=_zero_range, args=(buf, o, min(step, n - o)), daemon=True)
        th.start()
        threads.append(th)
    return buf, threads


class Simulation:
    """Fixed-step driver (llg.py:264-379), device resident."""

    CHUNK = 256        # max steps per device launch batch without an equilibrium stop
    CHUNK_EQ = 32      # ... with an equilibrium stop (bounds wasted queued work)
    PREFAULT_BYTES = 256 << 20   # fault in the final readback array during the run from this size
    STAGE_FIELD_BYTES = 256 << 20   # host bias fields per device chunk (callable spatial bias)

    def __init__(self, state: SimState, rhs: PartitionedRHS, ispec: IntegratorSpec,
                 sample_every: int = 1, sample_callback=None, energy_in_samples: bool = True):
        self.state = state
        self.rhs = rhs
        self.ispec = ispec
        self.sample_every = max(int(sample_every), 1)
        self.sample_callback = sample_callback
        self.energy_in_samples = energy_in_samples
        self._wall = 0.0
        if ispec.method == "mri-kw3":
            if not rhs.terms_in(FAST):
                raise ValueError("multirate stepping needs a non-empty fast partition")
            if not rhs.terms_in(SLOW_EXPLICIT):
                raise ValueError("multirate stepping needs a non-empty slow partition")
        grid, mat = state.m.grid, rhs.mat

        def renorm_hook(y):
            f = VectorField3(grid, y)
            renormalize(f, mat)
            return f.data

        self._hook = renorm_hook

    # ---- helpers -------------------------------------------------------------
    def _evals_per_step(self) -> dict:
        sp = self.ispec
        counts = {}
        for t in self.rhs.enabled_terms():
            if sp.method == "euler":
                counts[t] = 1
            elif sp.method == "rk4":
                counts[t] = 4
            else:
                counts[t] = fast_evals_per_step(sp.theta) if self.rhs.partition[t] == FAST else 3
        return counts

    def _sample_row_dev(self, ctx, state: SimState) -> dict:
        rhs = self.rhs
        mbar = np.zeros(3)
        L.check(ctx.call("mxb_state_mean", L.dptr(mbar)), "state_mean")
        row = {"t": state.t, "mx": mbar[0], "my": mbar[1], "mz": mbar[2],
               "e_demag": 0.0, "e_exch": 0.0, "e_anis": 0.0, "e_total": 0.0,
               "n_demag_evals": rhs.counters.get("demag", 0),
               "n_exch_evals": rhs.counters.get("exchange", 0), "wall_s": self._wall}
        if self.energy_in_samples:
            keep = []
            terms = tuple(x for x in ("demag", "bias") if x in rhs.enabled_terms())
            ts = rhs._terms_struct(terms)
            b = rhs._bias_struct(terms, state.t, None, keep)
            d = rhs._demag_dev._d.h if (rhs._demag_dev is not None and "demag" in terms) else None
            out = np.zeros(4)
            L.check(ctx.call("mxb_state_energies", d, C.byref(ts), C.byref(b), L.dptr(out)),
                    "state_energies")
            e = EnergyBreakdown(*(float(v) for v in out))
            row.update(e_demag=e.e_demag, e_exch=e.e_exch, e_anis=e.e_anis, e_total=e.e_total)
        return row

    def _sample_row_host(self, state: SimState) -> dict:
        mbar = mean_normalized(state.m, self.rhs.mat)
        row = {"t": state.t, "mx": mbar[0], "my": mbar[1], "mz": mbar[2],
               "e_demag": 0.0, "e_exch": 0.0, "e_anis": 0.0, "e_total": 0.0,
               "n_demag_evals": self.rhs.counters.get("demag", 0),
               "n_exch_evals": self.rhs.counters.get("exchange", 0), "wall_s": self._wall}
        if self.energy_in_samples:
            e = self.rhs.energies(state.t, state.m)
            row.update(e_demag=e.e_demag, e_exch=e.e_exch, e_anis=e.e_anis, e_total=e.e_total)
        return row

    def _n_total(self, stop: StopCondition, t0: float) -> int:
        sp = self.ispec
        n_total = None
        if stop.max_time is not None:
            n_total = max(int(round((stop.max_time - t0) / sp.dt)), 0)
        if stop.max_steps is not None:
            n_total = stop.max_steps if n_total is None else min(n_total, stop.max_steps)
        return n_total

    def _bias_times(self, t: float):
        """Times of the right-hand-side evaluations that read the bias in one
        step from t, in evaluation order (integrators.py:43-128)."""
        sp = self.ispec
        dt = sp.dt
        if sp.method == "euler":
            return [t]
        if sp.method == "rk4":
            half = 0.5 * dt
            return [t, t + half, t + half, t + dt]
        slow = self.rhs.partition.get("bias", SLOW_EXPLICIT) == SLOW_EXPLICIT
        nsub = substeps_per_phase(sp.theta)
        times = [t] if slow else []
        for ph in range(3):
            if not slow:
                span = _PHASE_WIDTH[ph] * dt
                t0 = t + KW3_C[ph] * dt
                h = span / nsub[ph]
                for s in range(nsub[ph]):
                    ts = t0 + s * h
                    times += [ts, ts + KW3_C[1] * h, ts + KW3_C[2] * h]
            if ph < 2 and slow:
                times.append(t + KW3_C[ph + 1] * dt)
        return times

    def run_until(self, stop: StopCondition) -> Trajectory:
        rhs, sp = self.rhs, self.ispec
        device = sp.method in ("euler", "rk4", "mri-kw3") and rhs._device_ok()
        b0 = None
        if device and rhs._bias is not None and not callable(rhs._bias):
            b0 = rhs.bias_at(0.0)
        if device:
            return self._run_device(stop, b0)
        return self._run_host(stop)

    # ---- device-resident loop ---------------------------------------------------
    def _run_device(self, stop: StopCondition, static_bias) -> Trajectory:
        state, rhs, sp = self.state, self.rhs, self.ispec
        mat = rhs.mat
        ctx = mat._ctx()
        traj = Trajectory()
        m0 = np.ascontiguousarray(state.m.data, dtype=np.float64)
        L.check(ctx.call("mxb_state_set", L.dptr(m0)), "state_set")
        grid = state.m.grid

        # the state read back at the end goes into a fresh array; for large grids
        # its pages are faulted in by host threads while the device steps, so
        # the final copy runs at copy speed instead of page-fault speed
        pf_on = os.environ.get("MXB_PREFAULT", "1") != "0"
        # (a sample callback pulls the state at every sample, so the buffer would
        # be used up at t = 0: prefault only runs without one)
        prefault = (_prefault((3,) + grid.shape) if pf_on and m0.nbytes >= self.PREFAULT_BYTES
                    and self.sample_callback is None else None)

        def pull():
            nonlocal prefault
            if prefault is not None:
                buf, threads = prefault
                prefault = None
                for th in threads:
                    th.join()
            else:
                buf = np.empty((3,) + grid.shape)
            L.check(ctx.call("mxb_state_get", L.dptr(buf)), "state_get")
            state.m = VectorField3(grid, buf)

        def emit():
            row = self._sample_row_dev(ctx, state)
            traj.samples.append(row)
            if self.sample_callback is not None:
                pull()
                self.sample_callback(state, row)

        t0, step0 = state.t, state.step
        n_total = self._n_total(stop, t0)
        start = time.perf_counter()
        wall_base = self._wall
        if mat.n_magnetic == 0:
            raise ValueError("mean_normalized: no magnetic cells (all Ms == 0)")
        emit()
        reason = "max_time" if stop.max_time is not None else "max_steps"
        if n_total is not None and stop.max_steps is not None and n_total == stop.max_steps:
            reason = "max_steps"
        terms = rhs.enabled_terms()
        ts = rhs._terms_struct(tuple(x for x in _ORDER if x in terms))
        evals = self._evals_per_step()
        d = rhs._demag_dev._d.h if rhs._demag_dev is not None else None
        eq = stop.equilibrium_tol
        keep = []
        args = L.RunArgs()
        args.method = {"rk4": L.RK4, "euler": L.EULER, "mri-kw3": L.MRI_KW3}[sp.method]
        args.theta = sp.theta
        args.fast_mask = sum(_BIT[x] for x in terms if rhs.partition[x] == FAST)
        args.renorm_each_stage = 1 if sp.renorm_each_stage else 0
        args.dt = sp.dt
        args.eq_tol = float(eq) if eq is not None else -1.0
        if static_bias is not None:
            if static_bias.shape == (3,):
                args.bias_vec = (C.c_double * 3)(*static_bias)
            else:
                f = np.ascontiguousarray(np.broadcast_to(static_bias, (3,) + grid.shape))
                keep.append(f)
                args.bias_field = L.dptr(f)
        k = 0
        equilibrated = False
        stats = L.RunStats()
        # a callable bias returning (3,nz,ny,nx) fields (reference llg.py:92-96,154-164;
        # scenario.build_bias returns one for every spatial expression): one field per
        # bias-reading evaluation is uploaded before that evaluation; chunks are sized
        # so the host fields of one chunk stay under STAGE_FIELD_BYTES
        probe = {}   # the shape probe at the first stage time is reused, not re-evaluated
        if callable(rhs._bias):
            first = self._bias_times(t0)
            if first:
                probe[first[0]] = rhs.bias_at(first[0])
        spatial = any(np.shape(v) != (3,) for v in probe.values())
        n_bias = max(len(self._bias_times(t0)), 1)

        def bias_at(tt):
            return probe.pop(tt) if tt in probe else rhs.bias_at(tt)

        field_chunk = max(1, self.STAGE_FIELD_BYTES // (n_bias * 24 * grid.n_cells))
        while k < n_total:
            to_sample = self.sample_every - (k % self.sample_every)
            chunk = min(n_total - k, to_sample, self.CHUNK_EQ if eq is not None else self.CHUNK)
            args.stage_bias_fields = None
            if spatial:
                chunk = min(chunk, field_chunk)
                flds = np.empty((chunk * n_bias, 3) + grid.shape)
                i = 0
                for s in range(chunk):
                    for tt in self._bias_times(t0 + (k + s) * sp.dt):
                        v = bias_at(tt)
                        flds[i] = v[:, None, None, None] if v.shape == (3,) else v
                        i += 1
                args.stage_bias_fields = L.dptr(flds)
                args.stage_bias = None
                keep_sbf = flds  # noqa: F841 (kept alive during the call)
            elif callable(rhs._bias):
                rows = []
                for s in range(chunk):
                    for tt in self._bias_times(t0 + (k + s) * sp.dt):
                        v = bias_at(tt)
                        if v.shape != (3,):
                            raise ValueError("a bias callable must return the same shape at every t")
                        rows.append(v)
                sb = np.ascontiguousarray(np.array(rows, dtype=np.float64))
                args.stage_bias = L.dptr(sb)
                keep_sb = sb  # noqa: F841 (kept alive during the call)
            else:
                args.stage_bias = None
            args.nsteps = chunk
            rc = ctx.call("mxb_run", d, C.byref(ts), C.byref(args), C.byref(stats))
            done = int(stats.steps_done)
            k += done
            state.t = t0 + k * sp.dt
            state.step = step0 + k
            for term, n in evals.items():
                rhs.counters[term] += n * done
            self._wall = wall_base + (time.perf_counter() - start)
            if rc == L.EBLOWUP:
                # the stage evaluations of the failed step were performed too
                for term, n in evals.items():
                    rhs.counters[term] += n
                pull()
                raise IntegrationBlowup(state.step + 1, state.t + sp.dt, float("inf")
                                        if stats.drift >= 1.79e308 else float(stats.drift))
            if rc == L.EDEAD:
                pull()
                _raise_dead(grid, int(stats.dead_flat))
            if rc != L.OK:
                # keep SimState consistent (t/step were advanced by steps_done)
                pull()
            L.check(rc, "run")
            traj.final_residual = float(stats.residual)
            equilibrated = stats.status == L.EQUILIBRATED
            if equilibrated:
                reason = "equilibrated"
            if k % self.sample_every == 0 or k == n_total or equilibrated:
                emit()
            if equilibrated:
                break
        if not equilibrated and eq is not None:
            reason = "not_converged"
        pull()
        traj.stop_reason = reason
        traj.counters = dict(rhs.counters)
        traj.wall_s = self._wall
        return traj

    # ---- host-orchestrated loop (plugin RHS / multirate) ----------------------
    def _advance(self, y, t):
        sp = self.ispec
        hook = self._hook if sp.renorm_each_stage else None
        if sp.method == "euler":
            return euler_step(y, t, sp.dt, self.rhs.rhs_total)
        if sp.method == "rk4":
            return rk4_step(y, t, sp.dt, self.rhs.rhs_total, hook)
        return mri_kw3_step(y, t, sp.dt, self.rhs.rhs_slow, self.rhs.rhs_fast, sp.theta, hook)

    def _run_host(self, stop: StopCondition) -> Trajectory:
        state, rhs, sp = self.state, self.rhs, self.ispec
        mat = rhs.mat
        traj = Trajectory()

        def emit():
            row = self._sample_row_host(state)
            traj.samples.append(row)
            if self.sample_callback is not None:
                self.sample_callback(state, row)

        t0, step0 = state.t, state.step
        n_total = self._n_total(stop, t0)
        start = time.perf_counter()
        wall_base = self._wall
        emit()
        prev_mean = mean_normalized(state.m, mat)
        reason = "max_time" if stop.max_time is not None else "max_steps"
        if n_total is not None and stop.max_steps is not None and n_total == stop.max_steps:
            reason = "max_steps"
        k = 0
        mask = mat.mask
        while k < n_total:
            y = self._advance(state.m.data, state.t)
            norms = np.sqrt(np.einsum("cijk,cijk->ijk", y, y))[mask]
            drift = float(np.max(np.abs(norms / mat.Ms[mask] - 1.0))) if norms.size else 0.0
            if not np.isfinite(drift) or drift > BLOWUP_DRIFT:
                raise IntegrationBlowup(state.step + 1, state.t + sp.dt,
                                        drift if np.isfinite(drift) else float("inf"))
            state.m = VectorField3(state.m.grid, y)
            renormalize(state.m, mat)
            k += 1
            state.t = t0 + k * sp.dt
            state.step = step0 + k
            self._wall = wall_base + (time.perf_counter() - start)
            cur_mean = mean_normalized(state.m, mat)
            traj.final_residual = float(np.max(np.abs(cur_mean - prev_mean)))
            equilibrated = (stop.equilibrium_tol is not None and
                            traj.final_residual < stop.equilibrium_tol)
            prev_mean = cur_mean
            if equilibrated:
                reason = "equilibrated"
            if k % self.sample_every == 0 or k == n_total or equilibrated:
                emit()
            if equilibrated:
                break
        else:
            if stop.equilibrium_tol is not None:
                reason = "not_converged"
        traj.stop_reason = reason
        traj.counters = dict(rhs.counters)
        traj.wall_s = self._wall
        return traj
