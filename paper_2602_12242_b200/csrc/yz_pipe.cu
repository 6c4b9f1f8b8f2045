// L2-resident y/z pipeline over kx planes (single GPU, 3-D, symmetric kernel).
//
// The 5-pass demag evaluation moves every intermediate through HBM; at 512^3
// the y/z middle (y forward, z fused, y inverse) alone is ~72 GB per
// evaluation although one kx plane of it (nz x py x 3 complex = 25 MB) fits in
// L2.  Here one persistent cooperative kernel processes work units of the hx
// kx-planes in dataflow order:
//   A(p, z)   y forward of row z of plane p : XP (HBM) -> slot[p % 3] [z][ky][c]
//   B(p, ky)  z forward * K * z inverse of column ky, in place in slot[p % 3]
//   C(p, z)   y inverse of row z            : slot[p % 3] -> XP (HBM, in place)
// with dependencies B(p, .) <- all A(p, .), C(p, .) <- all B(p, .) and
// A(p, z) <- C(p-3, z) (the slot row is reused three planes later).  The
// three slots (3 * nz * py * 48 B, 75 MB at 512^3) are meant to stay in L2, so
// HBM sees XP once each way plus the kernel spectra.
//
// Scheduling: an atomic ticket counter hands units out in rounds
//   round r = A(r) | B(r-1), first half of ky | C(r-2) | B(r-1), second half
// so that in steady state every dependency lies about one thousand tickets
// back (more than the units in flight): waits are rare.  Completion is
// counted per plane (A, B) and per slot row (C: a generation counter), polled
// with ld.acquire by one thread.  The per-unit round trips to L2 are kept off
// the critical path: the ticket after next is fetched early, the next unit's
// readiness is polled before the staging wait, and a unit's completion is
// signalled only after the next unit's staging wait (its stores have drained
// by then; immediately before any blocking wait, so signals cannot form a
// cycle between CTAs).  A wait longer than 2 s raises an abort word that makes
// every CTA leave: a scheduling bug cannot hang the device.
//
// Layouts: XP[kx][z][y][c] (plane-major x-pass output, written by
// k_r2c_fast with CH = CHP = 1), Kp[kx][ky'][kz'][6] real quarter spectra
// with ky' = min(ky, py-ky), kz' = min(kz, pz-kz) and the parity signs of
// XY/XZ/YZ (as k_quarterize).  k_yz_pipe uses the same register-resident
// radix-16 Stockham code (fft_fast.cuh) and twiddles as the 5-pass kernels, so
// both paths give identical results; k_yz_pipe_w (L = 1024, opt-in) uses the
// warp-per-line core of fft_warp.cuh.
#include <stdio.h>
#include <stdlib.h>
#include <type_traits>

#include "demag.cuh"
#include "tma.cuh"
#include "fft_fast.cuh"
#include "fft_warp.cuh"

#ifndef MXB_PIPE_W_CTAS
#define MXB_PIPE_W_CTAS 4
#endif
#ifndef MXB_PIPE_LATE_READ_WAIT
#define MXB_PIPE_LATE_READ_WAIT 1
#endif
#ifndef MXB_PIPE_TMA
#define MXB_PIPE_TMA 1
#endif
#ifndef MXB_PIPE_BULK
#define MXB_PIPE_BULK 1
#endif
#ifndef MXB_PIPE_DISCARD
#define MXB_PIPE_DISCARD 1
#endif
#ifndef MXB_PIPE_W_DIRECT_STORE
#define MXB_PIPE_W_DIRECT_STORE 0
#endif
// per-access L2 eviction hints in k_yz_pipe_w: 0 none; 1 slot ring evict_last,
// XP rows / kernel rows evict_first; 2 only the streams evict_first.
// Measured at 512^3 (profiles/round2_pipe_hints_ab.md): with the kz-pair kernel
// loads, 1 gives 20.13 ms per evaluation (DRAM 36.8 GB) vs 21.08 ms (49.1 GB)
#ifndef MXB_PIPE_HINTS
#define MXB_PIPE_HINTS 1
#endif
#ifndef MXB_PIPE_KPAIR      // B multiply: one kernel-entry load for kz and L - kz
#define MXB_PIPE_KPAIR 1
#endif
#ifndef MXB_PIPE_KPAIR_512  // the same in the L = 512 pair kernel (256^3: 16.28 -> 15.94 ms per step)
#define MXB_PIPE_KPAIR_512 1
#endif
#ifndef MXB_PIPE_DISCARD_LATE   // C units drop their slot row after the inverse FFT, not before
#define MXB_PIPE_DISCARD_LATE 0
#endif
#ifndef MXB_PIPE_SIGNAL_REL     // completion signals as red.release instead of fence + atomicAdd
#define MXB_PIPE_SIGNAL_REL 1
#endif
#ifndef MXB_PIPE_EARLY_READY // read the next unit's dependency counter during the current unit
#define MXB_PIPE_EARLY_READY 0
#endif
#ifndef MXB_PIPE_PF_NEXT     // L2 prefetch of the next A unit's XP row once its ticket is known
#define MXB_PIPE_PF_NEXT 0
#endif
#ifndef MXB_PIPE_PF_DIST     // ... of the A unit MXB_PIPE_PF_DIST tickets after the next (0: the next)
#define MXB_PIPE_PF_DIST 0
#endif
#ifndef MXB_PIPE_LATE_SIGNAL   // signal the previous unit mid-unit (after the next ticket), not before compute
#define MXB_PIPE_LATE_SIGNAL 0
#endif
#ifndef MXB_PIPE_SIGNAL_EARLY   // signal the previous unit between this unit's TMA issue and its wait
#define MXB_PIPE_SIGNAL_EARLY 1
#endif
#ifndef MXB_PIPE_NOBAR      // with the late signal: no CTA barrier after the staging wait
#define MXB_PIPE_NOBAR 0
#endif
#ifndef MXB_PIPE_KPRE       // B: first kernel entry loaded before the spectrum store + barrier
#define MXB_PIPE_KPRE 0
#endif
#ifndef MXB_PIPE_KPF_L1     // B multiply: L1 prefetch of the kernel entry this many iterations ahead
#define MXB_PIPE_KPF_L1 0
#endif
#ifndef MXB_PIPE_KROT       // B multiply: kernel entries loaded this many iterations ahead (0 = off)
#define MXB_PIPE_KROT 0
#endif
#ifndef MXB_PIPE_EARLY_ACQ  // next ticket + acquire of its dependency during this unit's staging wait
#define MXB_PIPE_EARLY_ACQ 0
#endif
#ifndef MXB_PIPE_SEEN       // skip re-acquiring a plane counter this CTA already saw complete
#define MXB_PIPE_SEEN 0
#endif
#ifndef MXB_PIPE_KUNROLL    // unroll of the B multiply's kernel-entry loop (loads of the next entry in flight)
#define MXB_PIPE_KUNROLL 1
#endif
#ifndef MXB_PIPE_HINT_K     // kernel-row loads with the evict_first hint too: same kernel time,
#define MXB_PIPE_HINT_K 1   // 27.7 instead of 36.9 GB of DRAM per launch -> more clock under the power cap
#endif
#if MXB_PIPE_HINTS
#define PIPE_POL_STREAM() policy_evict_first()
#if MXB_PIPE_HINTS == 1
#define PIPE_SLOT_HINTED 1
#define PIPE_POL_SLOT() policy_evict_last()
#else
#define PIPE_SLOT_HINTED 0
#endif
#endif

namespace mxb {

using namespace ff;

constexpr int kKUnroll = MXB_PIPE_KUNROLL;

struct PipeArgs {
    double2* XP;          // [hx][nz][ny][3], input and output (in place)
    double2* slot;        // 3 x [nz][L][3]
    const double* Kp;     // [hx][L/2+1][L/2+1][6]
    unsigned* sync;       // [ticket, abort, doneA[hx], doneB[hx], rowgen[3][n]], zeroed per launch
    int hx, n;            // planes; non-zero rows ny == nz == n
    double scale;
    int cplx;             // 1: Kp holds full complex spectra [hx][L][L][6] (double2), no symmetry assumed
    // z-slab decomposition (G ranks): XP is the all-to-all receive buffer
    // [g][hx][nzl][ny][3] -- row z of plane p lives in block g = z / nzl.  One
    // rank: nzl = n, a single block.
    int nzl;              // a power of two
    long long zjump;      // source block stride / nzl (elements per z of the block index)
};

// first element of row z (y line, 3 components) of plane p in XP
__device__ __forceinline__ long long xp_row(const PipeArgs& a, long long plane_xp, int p, int z, int rowlen) {
    const int zl = z & (a.nzl - 1);
    return (long long)(z - zl) * a.zjump + (long long)p * plane_xp + (long long)zl * rowlen;
}

// H = K M for one kz element with complex K (the reference's own tensor, whose
// spectra are not exactly real): k points at the six complex components
__device__ __forceinline__ void kmul_complex(const double2* __restrict__ k, double2& m0, double2& m1, double2& m2,
                                             double s) {
    const double2 kxx = __ldg(k), kxy = __ldg(k + 1), kxz = __ldg(k + 2);
    const double2 kyy = __ldg(k + 3), kyz = __ldg(k + 4), kzz = __ldg(k + 5);
    auto cm = [](double2 a, double2 b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); };
    auto ad = [](double2 a, double2 b, double2 c) { return make_double2(a.x + b.x + c.x, a.y + b.y + c.y); };
    const double2 h0 = ad(cm(kxx, m0), cm(kxy, m1), cm(kxz, m2));
    const double2 h1 = ad(cm(kxy, m0), cm(kyy, m1), cm(kyz, m2));
    const double2 h2 = ad(cm(kxz, m0), cm(kyz, m1), cm(kzz, m2));
    m0 = make_double2(h0.x * s, h0.y * s);
    m1 = make_double2(h1.x * s, h1.y * s);
    m2 = make_double2(h2.x * s, h2.y * s);
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_l2(double2* p, double2 v) {
    asm volatile("st.global.cg.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}

__device__ __forceinline__ void st_stream(double2* p, double2 v) {
    asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}


enum { U_NONE = 0, U_A = 1, U_B = 2, U_C = 3 };

struct Unit {
    int kind, plane, idx;
};

__device__ __forceinline__ int ky_of(int q, int L) {
    // pair ky with L - ky on neighbouring tickets: the shared K row is read once from HBM
    return q == 0 ? 0 : ((q & 1) ? (q + 1) / 2 : L - q / 2);
}

// ticket -> unit.  Round r (0 <= r <= hx+1) holds, in order:
//   A(r) [n, r < hx], B(r-1) q < L/2 [1 <= r <= hx], C(r-2) [n, r >= 2], B(r-1) q >= L/2
struct TicketMap {
    int hx, n, L;
    __device__ Unit operator()(long long k) const {
        const int h = L / 2;
        if (k < 0) return {U_NONE, 0, 0};
        // rounds 0 and 1
        if (k < n) return {U_A, 0, (int)k};
        k -= n;
        if (hx > 1) {
            if (k < n) return {U_A, 1, (int)k};
            k -= n;
        }
        if (k < L) return {U_B, 0, ky_of((int)k, L)};
        k -= L;
        // full rounds 2 .. hx-1
        const long long full = 2LL * n + L, nfull = hx > 2 ? hx - 2 : 0;
        if (k < nfull * full) {
            const int r = 2 + (int)(k / full);
            int o = (int)(k % full);
            if (o < n) return {U_A, r, o};
            o -= n;
            if (o < h) return {U_B, r - 1, ky_of(o, L)};
            o -= h;
            if (o < n) return {U_C, r - 2, o};
            return {U_B, r - 1, ky_of(h + o - n, L)};
        }
        k -= nfull * full;
        // round hx: B(hx-1) first half, C(hx-2), B(hx-1) second half (hx >= 2)
        if (hx >= 2) {
            if (k < h) return {U_B, hx - 1, ky_of((int)k, L)};
            k -= h;
            if (k < n) return {U_C, hx - 2, (int)k};
            k -= n;
            if (k < h) return {U_B, hx - 1, ky_of(h + (int)k, L)};
            k -= h;
        }
        // round hx+1: C(hx-1)
        if (k < n) return {U_C, hx - 1, (int)k};
        return {U_NONE, 0, 0};
    }
};

// dependency bookkeeping: doneA / doneB per plane, rowgen[slot][z] = number of
// C units that have drained slot row z (A(p, z) needs rowgen[p % 3][z] >= p / 3)
struct Sched {
    // one base pointer; the counters are derived on use (fewer live registers
    // across the unit loop of the FFT kernels)
    unsigned* base;
    int hx, n, L;
    int* halt;   // the run's halt word (null for a direct field evaluation)
    __device__ Sched(const PipeArgs& a, int L_, const int* halt_) :
        base(a.sync), hx(a.hx), n(a.n), L(L_), halt(const_cast<int*>(halt_)) {}
    __device__ unsigned* ticket() const { return base; }
    __device__ unsigned* abort_w() const { return base + 1; }
    __device__ unsigned* doneA() const { return base + 2; }
    __device__ unsigned* doneB() const { return base + 2 + hx; }
    __device__ unsigned* rowgen() const { return base + 2 + 2 * hx; }
    __device__ bool dep(const Unit& u, const unsigned** c, unsigned* target) const {
        if (u.kind == U_A) {
            if (u.plane < 3) return false;
            *c = rowgen() + (u.plane % 3) * n + u.idx;
            *target = (unsigned)(u.plane / 3);
        } else if (u.kind == U_B) {
            *c = doneA() + u.plane;
            *target = (unsigned)n;
        } else {
            *c = doneB() + u.plane;
            *target = (unsigned)L;
        }
        return true;
    }
    __device__ const unsigned* done_of(const Unit& u) const {
        if (u.kind == U_A) return doneA() + u.plane;
        if (u.kind == U_B) return doneB() + u.plane;
        return rowgen() + (u.plane % 3) * n + u.idx;
    }
    // thread 0: non-blocking readiness
    __device__ bool ready(const Unit& u) const {
        const unsigned* c;
        unsigned tg;
        return u.kind != U_NONE && (!dep(u, &c, &tg) || ld_acquire(c) >= tg);
    }
    // after a __syncthreads that follows the unit's stores; thread 0
    __device__ void signal(const Unit& u) const {
        if (threadIdx.x == 0) {
#if MXB_PIPE_SIGNAL_REL
            // one release reduction instead of a full fence and a relaxed atomic
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(done_of(u)) : "memory");
#else
            __threadfence();
            atomicAdd(const_cast<unsigned*>(done_of(u)), 1u);
#endif
        }
    }
    // CTA-wide wait for u's inputs.  Never blocks while holding an unsignalled
    // unit (deferred signals could otherwise form a cycle between CTAs);
    // pending is thread 0's.  Returns false on abort.
    // early: thread 0's relaxed read of u's counter, issued during the previous
    // unit (MXB_PIPE_EARLY_READY); if it already shows the target, the acquire
    // is a fence instead of another L2 round trip on the critical path
    // seen (thread 0, optional): the last plane whose A units (seen[0]) / B units
    // (seen[1]) this CTA has already observed complete with an acquire -- the
    // per-plane counters only grow and that acquire already ordered this CTA's
    // later reads after every producer, so further B / C units of the same
    // plane skip the load
    // acquired (thread 0): u's counter was already read with an acquire and showed
    // the target (MXB_PIPE_EARLY_ACQ) -- nothing to wait for, ordering established
    __device__ bool wait_ready(const Unit& u, int* flag, Unit& pending, unsigned early = 0u,
                               int* seen = nullptr, bool acquired = false) const {
        if (threadIdx.x == 0) {
            *flag = 1;
            const unsigned* c;
            unsigned tg;
            bool need = dep(u, &c, &tg) && !acquired;
            if (need && seen && ((u.kind == U_B && seen[0] == u.plane) || (u.kind == U_C && seen[1] == u.plane)))
                need = false;
            if (need && early >= tg) {
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
                need = false;
            }
            const bool observed = need;   // this unit's counter is read with an acquire below
            if (need && ld_acquire(c) < tg) {
                if (pending.kind != U_NONE) {
                    // the pending unit's bulk / TMA stores (async proxy) must have
                    // completed, not only read shared memory, before consumers see
                    // its signal (no-op for the cp.async-only kernels)
                    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                    signal(pending);
                    pending.kind = U_NONE;
                }
                const unsigned long long t0 = gtimer();
                while (ld_acquire(c) < tg) {
                    __nanosleep(32);
                    if (ld_acquire(abort_w())) { *flag = 0; break; }
                    if (gtimer() - t0 > 2000000000ull) {
                        printf("k_yz_pipe: wait timeout cta %d kind %d plane %d idx %d have %u need %u\n",
                               blockIdx.x, u.kind, u.plane, u.idx, ld_acquire(c), tg);
                        atomicExch(abort_w(), 1u);
                        // the run loop stops with MXB_ECUDA; a direct evaluation
                        // reports it from the abort word (DemagPlan::check_abort)
                        if (halt) atomicExch(halt, (int)MXB_ECUDA);
                        *flag = 0;
                        break;
                    }
                }
            }
            if (observed && seen && *flag) {
                if (u.kind == U_B) seen[0] = u.plane;
                if (u.kind == U_C) seen[1] = u.plane;
            }
        }
        __syncthreads();
        return *flag != 0;
    }
};

template <int L> struct PipeCfg {
    static constexpr int R = L >= 16 ? 16 : L;
    static constexpr int TPL = L / R;
    static constexpr int T = 3 * TPL;
    static constexpr int XE = smem_elems<L, R, 3>();   // >= 3 L
    static constexpr int SE = 3 * L;                    // staging: a unit's lines, or K rows
};

template <int L>
__global__ void __launch_bounds__(PipeCfg<L>::T, 2)
k_yz_pipe(PipeArgs a, const double2* __restrict__ tw, const int* __restrict__ halt) {
    if (halt && *halt) return;
    constexpr int R = PipeCfg<L>::R, TPL = PipeCfg<L>::TPL, T = PipeCfg<L>::T;
    constexpr int L2 = L / 2 + 1;
    extern __shared__ double2 sm[];
    __shared__ long long tk_sh;   // ticket of the unit after next
    __shared__ int flag;
    double2* X = sm;
    double2* S = sm + PipeCfg<L>::XE;
    const int n = a.n, hx = a.hx;
    const long long plane_xp = (long long)a.nzl * n * 3;       // XP elements per kx plane
    const long long slot_e = (long long)n * L * 3;         // slot elements
    const int b = threadIdx.x / TPL, t = threadIdx.x - (threadIdx.x / TPL) * TPL;
    const Sched sc(a, L, halt);
    const TicketMap tmap{hx, n, L};

    // unit inputs, staged in S with cp.async: A an XP row (HBM), B a slot
    // column (L2), C a slot row (L2); B also stages its K rows (HBM) over its
    // own forward FFT
    auto stage_in = [&](const Unit& u) {
        if (u.kind == U_A) {
            const double2* src = a.XP + xp_row(a, plane_xp, u.plane, u.idx, n * 3);
            for (int j = threadIdx.x; j < 3 * n; j += T) cp_async16(&S[j], src + j, true);
        } else if (u.kind == U_B) {
            const double2* col = a.slot + (long long)(u.plane % 3) * slot_e + (long long)u.idx * 3;
            for (int j = threadIdx.x; j < 3 * n; j += T) {
                const int z = j / 3, c = j - 3 * z;
                cp_async16(&S[j], col + (long long)z * L * 3 + c, true);
            }
        } else if (u.kind == U_C) {
            const double2* src = a.slot + (long long)(u.plane % 3) * slot_e + (long long)u.idx * L * 3;
            for (int j = threadIdx.x; j < 3 * L; j += T) cp_async16(&S[j], src + j, true);
        }
        cp_async_commit();
    };
    auto stage_k = [&](const Unit& u) {
        const int kyq = 2 * u.idx > L ? L - u.idx : u.idx;
        const double2* src = reinterpret_cast<const double2*>(a.Kp + ((long long)u.plane * L2 + kyq) * L2 * 6);
        for (int j = threadIdx.x; j < 3 * L2; j += T) cp_async16(&S[j], src + j, true);
        cp_async_commit();
    };

    // thread 0's private state: the unsignalled previous unit and the ticket
    // being fetched for the unit after next
    Unit pending{U_NONE, 0, 0};
    long long tk2 = -1;
    if (threadIdx.x == 0) {
        const long long t0 = atomicAdd(sc.ticket(), 1u);
        tk_sh = atomicAdd(sc.ticket(), 1u);
        flag = (int)t0;
    }
    __syncthreads();
    Unit cur = tmap(flag);
    Unit nxt = tmap(tk_sh);
    bool staged = false;

    while (cur.kind != U_NONE) {
        if (!staged) {
            if (!sc.wait_ready(cur, &flag, pending)) return;
            stage_in(cur);
        }
        // round trips issued now, consumed later: the ticket after next, and
        // (below) nxt's readiness
        bool nxt_ready = false;
        if (threadIdx.x == 0) {
            tk2 = atomicAdd(sc.ticket(), 1u);
            nxt_ready = sc.ready(nxt);
        }
        double2* slot = a.slot + (long long)(cur.plane % 3) * slot_e;
        const int nin = cur.kind == U_C ? L : n;
        double2 v[R];
        cp_async_wait_all();
        if (threadIdx.x == 0) {
            if (pending.kind != U_NONE) {
                sc.signal(pending);
                pending.kind = U_NONE;
            }
            flag = nxt_ready;
        }
        __syncthreads();
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const int e = t + m * TPL;
            v[m] = e < nin ? S[e * 3 + b] : make_double2(0.0, 0.0);
        }
        __syncthreads();
        const bool can_stage = flag != 0;
        bool staged_next = false;

        if (cur.kind == U_A) {
            // ---- y forward of row z = idx -> slot row
            if (can_stage) { stage_in(nxt); staged_next = true; }
            fft_core<L, R, 3, false, -1>(v, X, b, t, tw);
            __syncthreads();
#pragma unroll
            for (int i = 0; i < R; ++i) X[out_elem<L, R>(t, i) * 3 + b] = v[i];
            __syncthreads();
            double2* dst = slot + (long long)cur.idx * L * 3;
            for (int j = threadIdx.x; j < 3 * L; j += T) st_l2(dst + j, X[j]);
        } else if (cur.kind == U_B) {
            // ---- z forward * K * z inverse of column ky = idx, in place in the slot
            const int ky = cur.idx;
            stage_k(cur);
            fft_core<L, R, 3, false, -1>(v, X, b, t, tw);
            __syncthreads();
#pragma unroll
            for (int i = 0; i < R; ++i) X[out_elem<L, R>(t, i) * 3 + b] = v[i];
            cp_async_wait_all();
            __syncthreads();
            const bool fy = 2 * ky > L;
            const double s = a.scale;
            for (int kz = threadIdx.x; kz < L; kz += T) {
                const bool fz = 2 * kz > L;
                const int kzq = fz ? L - kz : kz;
                const double* k = reinterpret_cast<const double*>(S) + kzq * 6;
                const double2 m0 = X[kz * 3], m1 = X[kz * 3 + 1], m2 = X[kz * 3 + 2];
                const double kxx = k[0], kyy = k[3], kzz = k[5];
                const double kxy = fy ? -k[1] : k[1];
                const double kxz = fz ? -k[2] : k[2];
                const double kyz = (fy != fz) ? -k[4] : k[4];
                const double2 h0 = make_double2(kxx * m0.x + kxy * m1.x + kxz * m2.x,
                                                kxx * m0.y + kxy * m1.y + kxz * m2.y);
                const double2 h1 = make_double2(kxy * m0.x + kyy * m1.x + kyz * m2.x,
                                                kxy * m0.y + kyy * m1.y + kyz * m2.y);
                const double2 h2 = make_double2(kxz * m0.x + kyz * m1.x + kzz * m2.x,
                                                kxz * m0.y + kyz * m1.y + kzz * m2.y);
                X[kz * 3] = make_double2(h0.x * s, h0.y * s);
                X[kz * 3 + 1] = make_double2(h1.x * s, h1.y * s);
                X[kz * 3 + 2] = make_double2(h2.x * s, h2.y * s);
            }
            __syncthreads();
            if (can_stage) { stage_in(nxt); staged_next = true; }
#pragma unroll
            for (int m = 0; m < R; ++m) v[m] = X[(t + m * TPL) * 3 + b];
            fft_core<L, R, 3, false, 1>(v, X, b, t, tw);
            __syncthreads();
#pragma unroll
            for (int i = 0; i < R; ++i) {
                const int e = out_elem<L, R>(t, i);
                if (e < n) X[e * 3 + b] = v[i];
            }
            __syncthreads();
            double2* col = slot + (long long)ky * 3;
            for (int j = threadIdx.x; j < 3 * n; j += T) {
                const int z = j / 3, c = j - 3 * z;
                st_l2(col + (long long)z * L * 3 + c, X[j]);
            }
        } else {
            // ---- y inverse of row z = idx -> XP row (n of L kept)
            if (can_stage) { stage_in(nxt); staged_next = true; }
            fft_core<L, R, 3, false, 1>(v, X, b, t, tw);
            __syncthreads();
#pragma unroll
            for (int i = 0; i < R; ++i) {
                const int e = out_elem<L, R>(t, i);
                if (e < n) X[e * 3 + b] = v[i];
            }
            __syncthreads();
            double2* dst = a.XP + xp_row(a, plane_xp, cur.plane, cur.idx, n * 3);
            for (int j = threadIdx.x; j < 3 * n; j += T) st_stream(dst + j, X[j]);
        }
        if (threadIdx.x == 0) {
            tk_sh = tk2;
            pending = cur;
        }
        __syncthreads();
        cur = nxt;
        nxt = tmap(tk_sh);
        staged = staged_next;
    }
    if (threadIdx.x == 0 && pending.kind != U_NONE) sc.signal(pending);
}

// ---------------------------------------------------------------------------
// warp-FFT variant, L = 1024 (n = 512): one line per warp (fft_warp.cuh), the
// CTA is the component triple.  W (3 x 1024 = 48 KB) first stages the unit's
// lines (cp.async, natural [e][3] layout), then serves as the three warps'
// transpose tiles and B's component exchange; B reads its kernel rows through
// the read-only path.  48 KB and 168 registers give four CTAs (12 warps) per
// SM.  Zero-padded halves (A/B inputs, B/C outputs) are compile-time and fold
// away.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(96, MXB_PIPE_W_CTAS)
k_yz_pipe_w(PipeArgs a, const double2* __restrict__ tw, const int* __restrict__ halt,
            const __grid_constant__ CUtensorMap tmap_slot) {
    if (halt && *halt) return;
    constexpr int L = 1024, N = 512, L2 = L / 2 + 1;
    extern __shared__ __align__(128) double2 sm[];
    __shared__ long long next_ticket;
    __shared__ int flag;
    __shared__ alignas(8) unsigned long long mbar;           // bulk row copies (A, C)
    double2* W = sm;                                        // 3 x 1024
    // kernel rows are read through the read-only path in the multiply (a
    // warp's 32 consecutive kz rows are 1.5 KB contiguous)
    const double2* __restrict__ Kp2 = reinterpret_cast<const double2*>(a.Kp);
    const int hx = a.hx;
    const long long plane_xp = (long long)a.nzl * N * 3, slot_e = (long long)N * L * 3;
    const int c = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double2* Wc = W + c * L;
    const Sched sc(a, L, halt);
    const TicketMap tmap{hx, N, L};
#if MXB_PIPE_SEEN
    int seen[2] = {-1, -1};   // thread 0: planes whose A / B units are known complete
#endif
#if MXB_PIPE_EARLY_READY
    unsigned early = 0u;   // thread 0: the next unit's dependency counter, read during this unit
    auto early_read = [&](long long t) -> unsigned {
        const Unit nu = tmap(t);
        const unsigned* cc;
        unsigned tg;
        return sc.dep(nu, &cc, &tg) ? ld_relaxed(cc) : 0u;
    };
#endif
#if MXB_PIPE_PF_NEXT
    // thread 0, once the next ticket is known: an A unit's XP row comes from
    // DRAM -- start pulling it into L2 while this unit finishes
    auto prefetch_next_a = [&](long long t) {
        const Unit nu = tmap(t + MXB_PIPE_PF_DIST);
        if (nu.kind == U_A)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                             a.XP + xp_row(a, plane_xp, nu.plane, nu.idx, N * 3)),
                         "r"(3 * N * 16)
                         : "memory");
    };
#endif

    auto stage = [&](const Unit& u) {
        double2* slot = a.slot + (long long)(u.plane % 3) * slot_e;
#if MXB_PIPE_LATE_READ_WAIT
        // the previous unit's store from W must have read it before this
        // unit's input lands in W (thread 0 issues both)
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#endif
        if (u.kind == U_A) {
#if MXB_PIPE_BULK
            if (threadIdx.x == 0) {
#if MXB_PIPE_HINTS
                bulk_g2s_hint(W, a.XP + xp_row(a, plane_xp, u.plane, u.idx, N * 3), 3 * N * 16, &mbar,
                              PIPE_POL_STREAM());
#else
                bulk_g2s(W, a.XP + xp_row(a, plane_xp, u.plane, u.idx, N * 3), 3 * N * 16, &mbar);
#endif
            }
#else
            const double2* src = a.XP + xp_row(a, plane_xp, u.plane, u.idx, N * 3);
            for (int j = threadIdx.x; j < 3 * N; j += 96) cp_async16(&W[j], src + j, true);
#endif
        } else if (u.kind == U_B) {
#if MXB_PIPE_TMA
            if (threadIdx.x == 0) {
                // the column, z 0..255 and 256..511, as two tensor boxes -> W [z][c]
                asm volatile("fence.proxy.async.global;" ::: "memory");
                mbar_expect(&mbar, 2 * 256 * 48);
                const int y0 = (u.plane % 3) * N;
#if MXB_PIPE_HINTS && PIPE_SLOT_HINTED
                const unsigned long long ps = PIPE_POL_SLOT();
                tma_load_2d_hint(W, &tmap_slot, u.idx * 6, y0, &mbar, ps);
                tma_load_2d_hint(W + 768, &tmap_slot, u.idx * 6, y0 + 256, &mbar, ps);
#else
                tma_load_2d(W, &tmap_slot, u.idx * 6, y0, &mbar);
                tma_load_2d(W + 768, &tmap_slot, u.idx * 6, y0 + 256, &mbar);
#endif
            }
#else
            const double2* col = slot + (long long)u.idx * 3;
            for (int j = threadIdx.x; j < 3 * N; j += 96) {
                const int z = j / 3, cc = j - 3 * z;
                cp_async16(&W[j], col + (long long)z * L * 3 + cc, true);
            }
#endif
            if (threadIdx.x == 0) {
                // pull the unit's kernel row (L2 x 48 B) into L2 over the forward FFT;
                // the multiply reads it through the read-only path
                if (a.cplx) {
                    const double* kr = a.Kp + ((long long)u.plane * L + u.idx) * L * 12;
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(kr), "r"(L * 96) : "memory");
                } else {
                    const int kyq = 2 * u.idx > L ? L - u.idx : u.idx;
                    const double* kr = a.Kp + ((long long)u.plane * L2 + kyq) * L2 * 6;
#if MXB_PIPE_HINTS
                    prefetch_l2_hint(kr, L2 * 48, PIPE_POL_STREAM());
#else
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(kr), "r"(L2 * 48) : "memory");
#endif
                }
            }
        } else {
#if MXB_PIPE_BULK
            if (threadIdx.x == 0) {
                asm volatile("fence.proxy.async.global;" ::: "memory");
#if MXB_PIPE_HINTS
                bulk_g2s_hint(W, slot + (long long)u.idx * L * 3, 3 * L * 16, &mbar, PIPE_POL_STREAM());
#else
                bulk_g2s(W, slot + (long long)u.idx * L * 3, 3 * L * 16, &mbar);
#endif
            }
#else
            const double2* src = slot + (long long)u.idx * L * 3;
            for (int j = threadIdx.x; j < 3 * L; j += 96) cp_async16(&W[j], src + j, true);
#endif
        }
        cp_async_commit();
    };
    unsigned mphase = 0;
    // wait for the staged input of u (cp.async group and, for A and C, the bulk copy)
    auto stage_wait = [&](const Unit& u) {
        cp_async_wait_all();
#if MXB_PIPE_BULK
        if (u.kind != U_B || MXB_PIPE_TMA) {
            mbar_wait(&mbar, mphase);
            mphase ^= 1u;
        }
#endif
    };
    // registers (lane j holds e = j + 32 k in v[p32(k)], k < NK) -> W natural [e][3]
    // -> contiguous 16-byte stores of the first ne elements (whole sectors per warp)
    auto store_rows = [&](double2 (&v)[32], auto nk_tag, double2* dst, int ne, bool stream, int lane) {
        constexpr int NK = decltype(nk_tag)::value;
        __syncthreads();   // every warp is done with its transpose tile
#pragma unroll
        for (int k = 0; k < NK; ++k) W[(lane + 32 * k) * 3 + c] = v[fw::p32(k)];
#if MXB_PIPE_TMA
        // one bulk store of the contiguous row (the next unit stages into W, so
        // the store must have read it before the end-of-unit barrier)
#if !MXB_PIPE_HINTS
        (void)stream;
#endif
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
#if MXB_PIPE_HINTS
            if (stream)
                bulk_s2g_hint(dst, W, 3 * ne * 16, PIPE_POL_STREAM());
#if PIPE_SLOT_HINTED
            else
                bulk_s2g_hint(dst, W, 3 * ne * 16, PIPE_POL_SLOT());
#else
            else
                bulk_s2g(dst, W, 3 * ne * 16);
#endif
#else
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                         "r"(smem_u32(W)), "r"(3 * ne * 16)
                         : "memory");
#endif
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
#if !MXB_PIPE_LATE_READ_WAIT
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#endif
        }
#else
        __syncthreads();
        if (stream)
            for (int j = threadIdx.x; j < 3 * ne; j += 96) st_stream(dst + j, W[j]);
        else
            for (int j = threadIdx.x; j < 3 * ne; j += 96) st_l2(dst + j, W[j]);
#endif
    };

    if (threadIdx.x == 0) {
        next_ticket = atomicAdd(sc.ticket(), 1u);
#if MXB_PIPE_BULK
        mbar_init(&mbar);
#endif
    }
    __syncthreads();
    Unit cur = tmap(next_ticket);
#if MXB_PIPE_EARLY_ACQ
    bool early_ok = false;   // thread 0: cur's dependency already acquired as complete
#endif
    // completion of the previous unit is signalled after this unit's staging
    // wait (its stores have drained by then), or before blocking
    Unit pending{U_NONE, 0, 0};

    while (cur.kind != U_NONE) {
#if MXB_PIPE_EARLY_READY
        if (!sc.wait_ready(cur, &flag, pending, early)) return;
        early = 0u;
#elif MXB_PIPE_SEEN
        if (!sc.wait_ready(cur, &flag, pending, 0u, seen)) return;
#elif MXB_PIPE_EARLY_ACQ
        if (!sc.wait_ready(cur, &flag, pending, 0u, nullptr, early_ok)) return;
        early_ok = false;
#else
        if (!sc.wait_ready(cur, &flag, pending)) return;
#endif
        stage(cur);
#if MXB_PIPE_SIGNAL_EARLY
        // the previous unit's completion while this unit's input is in flight: the
        // wait for its stores to complete overlaps the TMA latency, and consumers
        // see the signal one staging wait earlier
        if (pending.kind != U_NONE) {
            if (threadIdx.x == 0) {
                asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
                asm volatile("fence.proxy.async.global;" ::: "memory");
            }
            sc.signal(pending);
            pending.kind = U_NONE;
        }
#endif
#if MXB_PIPE_EARLY_ACQ
        // thread 0, while this unit's input is in flight: the next ticket, and an
        // acquire read of its dependency counter (both latencies overlap the
        // staging wait instead of the FFT and the next unit's start); a single
        // read, never a blocking wait
        if (threadIdx.x == 0) {
            next_ticket = atomicAdd(sc.ticket(), 1u);
            const Unit nu = tmap(next_ticket);
            early_ok = nu.kind != U_NONE && sc.ready(nu);
        }
#endif
        stage_wait(cur);
#if !MXB_PIPE_LATE_SIGNAL
        if (pending.kind != U_NONE) {
            if (threadIdx.x == 0) {
                // a B unit's column went out as TMA stores: complete them first
                asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
                asm volatile("fence.proxy.async.global;" ::: "memory");
            }
            sc.signal(pending);
            pending.kind = U_NONE;
        }
#endif
#if !(MXB_PIPE_LATE_SIGNAL && MXB_PIPE_NOBAR)
        // (with the late signal nothing here needs the CTA: every thread has waited
        // for the staged input on the mbarrier itself)
        __syncthreads();
#endif
        double2* slot = a.slot + (long long)(cur.plane % 3) * slot_e;
#if MXB_PIPE_DISCARD && !MXB_PIPE_DISCARD_LATE
        if (cur.kind == U_C) {
            // the slot row is dead until A(p+3, z) rewrites it: drop its L2 lines
            // without writing them back (48 KB = 384 lines of 128 B)
            char* row = reinterpret_cast<char*>(slot + (long long)cur.idx * L * 3);
            for (int j = threadIdx.x; j < 3 * L * 16 / 128; j += 96)
                asm volatile("discard.global.L2 [%0], 128;" ::"l"(row + (size_t)j * 128) : "memory");
        }
#endif
        // one forward FFT instance (A, B: zero-padded inputs) and one inverse
        // instance (B, C: half of the outputs kept) -- four inlined FFT bodies
        // overflowed the instruction cache
        double2 v[32];
        if (cur.kind == U_C) {
#pragma unroll
            for (int m = 0; m < 32; ++m) v[m] = W[(lane + 32 * m) * 3 + c];
        } else {
#pragma unroll
            for (int m = 0; m < 32; ++m) v[m] = m < 16 ? W[(lane + 32 * m) * 3 + c] : make_double2(0.0, 0.0);
        }
        __syncthreads();   // W becomes the transpose tiles
        bool inverse = cur.kind == U_C;
        if (cur.kind != U_C) {
            fw::fft1024<-1, MXB_HALF_IN != 0>(v, Wc, lane, tw);
            if (threadIdx.x == 0) {
#if !MXB_PIPE_EARLY_ACQ
                next_ticket = atomicAdd(sc.ticket(), 1u);
#endif
#if MXB_PIPE_PF_NEXT
                prefetch_next_a(next_ticket);
#endif
#if MXB_PIPE_EARLY_READY
                early = early_read(next_ticket);
#endif
#if MXB_PIPE_LATE_SIGNAL
                // the previous unit's completion, off the critical path: its bulk /
                // TMA stores finished long ago; no blocking wait lies between
                if (pending.kind != U_NONE) {
                    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                    sc.signal(pending);
                    pending.kind = U_NONE;
                }
#endif
            }
            if (cur.kind == U_A) {
                // ---- y forward of row z = idx -> slot row [ky][c]
#if MXB_PIPE_W_DIRECT_STORE
                double2* dst = slot + (long long)cur.idx * L * 3 + c;
#pragma unroll
                for (int k = 0; k < 32; ++k) st_l2(dst + (long long)(lane + 32 * k) * 3, v[fw::p32(k)]);
#else
                store_rows(v, std::integral_constant<int, 32>{}, slot + (long long)cur.idx * L * 3, L, false, lane);
#endif
            } else {
                // ---- B: * K between the z forward and z inverse of column ky = idx
                const int ky = cur.idx;
#if MXB_PIPE_KPRE && MXB_PIPE_KPAIR
                // this thread's first kernel entry (q = threadIdx.x <= L/2), loaded before
                // the spectrum goes to shared memory: its latency overlaps the stores and
                // the barrier
                const double2* kpre = Kp2 + ((long long)cur.plane * L2 + (2 * ky > L ? L - ky : ky)) * L2 * 3 +
                                      threadIdx.x * 3;
                const double2 pre01 = __ldg(kpre), pre23 = __ldg(kpre + 1), pre45 = __ldg(kpre + 2);
#endif
                __syncwarp();
#pragma unroll
                for (int k = 0; k < 32; ++k) Wc[lane + 32 * k] = v[fw::p32(k)];
                __syncthreads();
                const bool fy = 2 * ky > L;
                const double s = a.scale;
                if (a.cplx) {
                    const double2* krow = Kp2 + ((long long)cur.plane * L + ky) * L * 6;
                    for (int kz = threadIdx.x; kz < L; kz += 96)
                        kmul_complex(krow + kz * 6, W[kz], W[L + kz], W[2 * L + kz], s);
                }
                const double2* krow = Kp2 + ((long long)cur.plane * L2 + (fy ? L - ky : ky)) * L2 * 3;
#if MXB_PIPE_HINTS && MXB_PIPE_HINT_K
                const unsigned long long pk = PIPE_POL_STREAM();
#endif
                // each thread owns whole kz rows (all 3 components), in place in W
#if MXB_PIPE_KPAIR
                // kz and L - kz share the parity-reduced entry kz' = min(kz, L - kz):
                // each entry is loaded once and applied to both (sign flip of XZ, YZ)
#if MXB_PIPE_KROT
                // kernel entries rotated through registers: the loads of the entry
                // MXB_PIPE_KROT iterations ahead are in flight during this one's updates
                constexpr int KD = MXB_PIPE_KROT;
                double2 kq[KD][3];
                {
                    const int q0 = a.cplx ? L : (int)threadIdx.x;
#pragma unroll
                    for (int d = 0; d < KD; ++d) {
                        const int qd = q0 + 96 * d;
                        if (qd <= L / 2) {
                            const double2* kr = krow + qd * 3;
#if MXB_PIPE_HINTS && MXB_PIPE_HINT_K
                            kq[d][0] = ldg_hint(kr, pk); kq[d][1] = ldg_hint(kr + 1, pk); kq[d][2] = ldg_hint(kr + 2, pk);
#else
                            kq[d][0] = __ldg(kr); kq[d][1] = __ldg(kr + 1); kq[d][2] = __ldg(kr + 2);
#endif
                        }
                    }
                }
#endif
#if MXB_PIPE_KUNROLL > 1
#pragma unroll(kKUnroll)
#endif
                for (int q = a.cplx ? L : threadIdx.x; q <= L / 2; q += 96) {
                    const double2* kr = krow + q * 3;
#if MXB_PIPE_KPF_L1
                    // the entry MXB_PIPE_KPF_L1 iterations ahead into L1 (no registers held)
                    if (q + 96 * MXB_PIPE_KPF_L1 <= L / 2) {
                        const char* pn = reinterpret_cast<const char*>(kr + 96 * MXB_PIPE_KPF_L1 * 3);
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(pn));
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(pn + 47));
                    }
#endif
#if MXB_PIPE_KROT
                    const double2 q01 = kq[0][0], q23 = kq[0][1], q45 = kq[0][2];
#pragma unroll
                    for (int d = 0; d + 1 < KD; ++d) {
                        kq[d][0] = kq[d + 1][0]; kq[d][1] = kq[d + 1][1]; kq[d][2] = kq[d + 1][2];
                    }
                    if (q + 96 * KD <= L / 2) {
                        const double2* kn = kr + 96 * KD * 3;
#if MXB_PIPE_HINTS && MXB_PIPE_HINT_K
                        kq[KD - 1][0] = ldg_hint(kn, pk); kq[KD - 1][1] = ldg_hint(kn + 1, pk);
                        kq[KD - 1][2] = ldg_hint(kn + 2, pk);
#else
                        kq[KD - 1][0] = __ldg(kn); kq[KD - 1][1] = __ldg(kn + 1); kq[KD - 1][2] = __ldg(kn + 2);
#endif
                    }
#elif MXB_PIPE_KPRE
                    double2 q01, q23, q45;
                    if (q == (int)threadIdx.x) {
                        q01 = pre01; q23 = pre23; q45 = pre45;
                    } else {
#if MXB_PIPE_HINTS && MXB_PIPE_HINT_K
                        q01 = ldg_hint(kr, pk); q23 = ldg_hint(kr + 1, pk); q45 = ldg_hint(kr + 2, pk);
#else
                        q01 = __ldg(kr); q23 = __ldg(kr + 1); q45 = __ldg(kr + 2);
#endif
                    }
#elif MXB_PIPE_HINTS && MXB_PIPE_HINT_K
                    const double2 q01 = ldg_hint(kr, pk), q23 = ldg_hint(kr + 1, pk), q45 = ldg_hint(kr + 2, pk);
#else
                    const double2 q01 = __ldg(kr), q23 = __ldg(kr + 1), q45 = __ldg(kr + 2);
#endif
                    const double kxx = q01.x, kyy = q23.y, kzz = q45.y;
                    const double kxy = fy ? -q01.y : q01.y;
                    auto apply = [&](int kz, double kxz, double kyz) {
                        const double2 m0 = W[kz], m1 = W[L + kz], m2 = W[2 * L + kz];
                        const double2 h0 = make_double2(kxx * m0.x + kxy * m1.x + kxz * m2.x,
                                                        kxx * m0.y + kxy * m1.y + kxz * m2.y);
                        const double2 h1 = make_double2(kxy * m0.x + kyy * m1.x + kyz * m2.x,
                                                        kxy * m0.y + kyy * m1.y + kyz * m2.y);
                        const double2 h2 = make_double2(kxz * m0.x + kyz * m1.x + kzz * m2.x,
                                                        kxz * m0.y + kyz * m1.y + kzz * m2.y);
                        W[kz] = make_double2(h0.x * s, h0.y * s);
                        W[L + kz] = make_double2(h1.x * s, h1.y * s);
                        W[2 * L + kz] = make_double2(h2.x * s, h2.y * s);
                    };
                    const double kyz0 = fy ? -q45.x : q45.x;
                    apply(q, q23.x, kyz0);
                    if (q != 0 && q != L / 2) apply(L - q, -q23.x, -kyz0);
                }
#else
                for (int kz = a.cplx ? L : threadIdx.x; kz < L; kz += 96) {
                    const bool fz = 2 * kz > L;
                    const double2* kr = krow + (fz ? L - kz : kz) * 3;
#if MXB_PIPE_HINTS && MXB_PIPE_HINT_K
                    const double2 q01 = ldg_hint(kr, pk), q23 = ldg_hint(kr + 1, pk), q45 = ldg_hint(kr + 2, pk);
#else
                    const double2 q01 = __ldg(kr), q23 = __ldg(kr + 1), q45 = __ldg(kr + 2);
#endif
                    const double kxx = q01.x, kyy = q23.y, kzz = q45.y;
                    const double kxy = fy ? -q01.y : q01.y;
                    const double kxz = fz ? -q23.x : q23.x;
                    const double kyz = (fy != fz) ? -q45.x : q45.x;
                    const double2 m0 = W[kz], m1 = W[L + kz], m2 = W[2 * L + kz];
                    const double2 h0 = make_double2(kxx * m0.x + kxy * m1.x + kxz * m2.x,
                                                    kxx * m0.y + kxy * m1.y + kxz * m2.y);
                    const double2 h1 = make_double2(kxy * m0.x + kyy * m1.x + kyz * m2.x,
                                                    kxy * m0.y + kyy * m1.y + kyz * m2.y);
                    const double2 h2 = make_double2(kxz * m0.x + kyz * m1.x + kzz * m2.x,
                                                    kxz * m0.y + kyz * m1.y + kzz * m2.y);
                    W[kz] = make_double2(h0.x * s, h0.y * s);
                    W[L + kz] = make_double2(h1.x * s, h1.y * s);
                    W[2 * L + kz] = make_double2(h2.x * s, h2.y * s);
                }
#endif
                __syncthreads();
#pragma unroll
                for (int m = 0; m < 32; ++m) v[m] = Wc[lane + 32 * m];
                __syncthreads();   // all reads of W done before the tiles are reused
                inverse = true;
            }
        }
        if (inverse) {
            fw::fft1024<1>(v, Wc, lane, tw);
#if MXB_PIPE_DISCARD && MXB_PIPE_DISCARD_LATE
            if (cur.kind == U_C) {
                char* row = reinterpret_cast<char*>(slot + (long long)cur.idx * L * 3);
                for (int j = threadIdx.x; j < 3 * L * 16 / 128; j += 96)
                    asm volatile("discard.global.L2 [%0], 128;" ::"l"(row + (size_t)j * 128) : "memory");
            }
#endif
            if (cur.kind == U_C) {
                // ---- y inverse of row z = idx -> XP row (n of L kept)
                if (threadIdx.x == 0) {
#if !MXB_PIPE_EARLY_ACQ
                    next_ticket = atomicAdd(sc.ticket(), 1u);
#endif
#if MXB_PIPE_PF_NEXT
                    prefetch_next_a(next_ticket);
#endif
#if MXB_PIPE_EARLY_READY
                    early = early_read(next_ticket);
#endif
#if MXB_PIPE_LATE_SIGNAL
                    // the previous unit's completion, off the critical path: its bulk /
                    // TMA stores finished long ago; no blocking wait lies between
                    if (pending.kind != U_NONE) {
                        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                        sc.signal(pending);
                        pending.kind = U_NONE;
                    }
#endif
                }
#if MXB_PIPE_W_DIRECT_STORE
                double2* dst = a.XP + xp_row(a, plane_xp, cur.plane, cur.idx, N * 3) + c;
#pragma unroll
                for (int k = 0; k < 16; ++k) st_stream(dst + (long long)(lane + 32 * k) * 3, v[fw::p32(k)]);
#else
                store_rows(v, std::integral_constant<int, 16>{}, a.XP + xp_row(a, plane_xp, cur.plane, cur.idx, N * 3),
                           N, true, lane);
#endif
            } else {
                // ---- B: the first n of the inverse column back into the slot
                __syncthreads();
#pragma unroll
                for (int k = 0; k < 16; ++k) W[(lane + 32 * k) * 3 + c] = v[fw::p32(k)];
#if MXB_PIPE_TMA
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncthreads();
                if (threadIdx.x == 0) {
                    const int y0 = (cur.plane % 3) * N;
#if MXB_PIPE_HINTS && PIPE_SLOT_HINTED
                    const unsigned long long ps = PIPE_POL_SLOT();
                    tma_store_2d_hint(&tmap_slot, cur.idx * 6, y0, W, ps);
                    tma_store_2d_hint(&tmap_slot, cur.idx * 6, y0 + 256, W + 768, ps);
#else
                    tma_store_2d(&tmap_slot, cur.idx * 6, y0, W);
                    tma_store_2d(&tmap_slot, cur.idx * 6, y0 + 256, W + 768);
#endif
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    // W is staged into by the next unit: the stores must have read it
                    // (waited for in the next stage(), or here)
#if !MXB_PIPE_LATE_READ_WAIT
                    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#endif
                }
#else
                __syncthreads();
                double2* col = slot + (long long)cur.idx * 3;
                for (int j = threadIdx.x; j < 3 * N; j += 96) {
                    const int z = j / 3, cc = j - 3 * z;
                    st_l2(col + (long long)z * L * 3 + cc, W[j]);
                }
#endif
            }
        }
        __syncthreads();
        pending = cur;
        cur = tmap(next_ticket);
    }
    if (threadIdx.x == 0) {
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    if (pending.kind != U_NONE) sc.signal(pending);
}



// ---------------------------------------------------------------------------
// prefetching variant of k_yz_pipe_w (opt-in, MXB_PIPE_PREFETCH=1): three CTAs
// per SM, each with a 24.6 KB side buffer Q into which the NEXT unit's input is
// staged by TMA while the current unit computes -- A rows and B columns fit in
// Q; C rows (49 KB) still stage into W synchronously.  Tickets are fetched two
// ahead so the next unit is known at the start of the current one.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(96, 3)
k_yz_pipe_wq(PipeArgs a, const double2* __restrict__ tw, const int* __restrict__ halt,
             const __grid_constant__ CUtensorMap tmap_slot) {
    if (halt && *halt) return;
    constexpr int L = 1024, N = 512, L2 = L / 2 + 1;
    extern __shared__ __align__(128) double2 sm[];
    __shared__ long long tk_sh;
    __shared__ int flag, qflag;
    __shared__ alignas(8) unsigned long long mbar, mbq;
    double2* W = sm;              // 3 x 1024: staging (C, unprefetched units), tiles, exchange
    double2* Q = sm + 3 * L;      // 3 x 512: the next A / B unit's input
    const double2* __restrict__ Kp2 = reinterpret_cast<const double2*>(a.Kp);
    const int hx = a.hx;
    const long long plane_xp = (long long)a.nzl * N * 3, slot_e = (long long)N * L * 3;
    const int c = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double2* Wc = W + c * L;
    const Sched sc(a, L, halt);
    const TicketMap tmap{hx, N, L};

    // thread 0: issue the staging of u into dst (A and B only into Q; any into W)
    auto issue = [&](const Unit& u, double2* dst, unsigned long long* mb) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        if (u.kind == U_A) {
            bulk_g2s(dst, a.XP + xp_row(a, plane_xp, u.plane, u.idx, N * 3), 3 * N * 16, mb);
        } else if (u.kind == U_B) {
            mbar_expect(mb, 2 * 256 * 48);
            const int y0 = (u.plane % 3) * N;
            tma_load_2d(dst, &tmap_slot, u.idx * 6, y0, mb);
            tma_load_2d(dst + 768, &tmap_slot, u.idx * 6, y0 + 256, mb);
            const int kyq = 2 * u.idx > L ? L - u.idx : u.idx;
            const double* kr = a.Kp + ((long long)u.plane * L2 + kyq) * L2 * 6;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(kr), "r"(L2 * 48) : "memory");
        } else {
            const double2* slot = a.slot + (long long)(u.plane % 3) * slot_e;
            bulk_g2s(dst, slot + (long long)u.idx * L * 3, 3 * L * 16, mb);
        }
    };
    auto bulk_store = [&](double2* dst, int nelem) {   // thread 0, after fence + barrier
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(W)),
                     "r"(nelem * 16)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    };

    Unit pending{U_NONE, 0, 0};
    long long tk2 = -1;
    if (threadIdx.x == 0) {
        mbar_init(&mbar);
        mbar_init(&mbq);
        flag = (int)atomicAdd(sc.ticket(), 1u);
        tk_sh = atomicAdd(sc.ticket(), 1u);
    }
    __syncthreads();
    Unit cur = tmap(flag);
    Unit nxt = tmap(tk_sh);
    unsigned mph = 0, mpq = 0;
    bool in_q = false;   // cur's input was prefetched into Q

    while (cur.kind != U_NONE) {
        if (!in_q) {
            if (!sc.wait_ready(cur, &flag, pending)) return;
            if (threadIdx.x == 0) issue(cur, W, &mbar);
        }
        bool nxt_ready = false;
        if (threadIdx.x == 0) {
            tk2 = atomicAdd(sc.ticket(), 1u);
            nxt_ready = (nxt.kind == U_A || nxt.kind == U_B) && sc.ready(nxt);
        }
        if (in_q) {
            mbar_wait(&mbq, mpq);
            mpq ^= 1u;
        } else {
            mbar_wait(&mbar, mph);
            mph ^= 1u;
        }
        if (threadIdx.x == 0) {
            if (pending.kind != U_NONE) {
                asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
                asm volatile("fence.proxy.async.global;" ::: "memory");
                sc.signal(pending);
                pending.kind = U_NONE;
            }
            qflag = nxt_ready;
        }
        __syncthreads();
        const double2* src = in_q ? Q : W;
        double2 v[32];
        if (cur.kind == U_C) {
#pragma unroll
            for (int m = 0; m < 32; ++m) v[m] = src[(lane + 32 * m) * 3 + c];
        } else {
#pragma unroll
            for (int m = 0; m < 32; ++m) v[m] = m < 16 ? src[(lane + 32 * m) * 3 + c] : make_double2(0.0, 0.0);
        }
        __syncthreads();   // W and Q are free: prefetch the next unit into Q
        const bool staged_next = qflag != 0;
        if (staged_next && threadIdx.x == 0) issue(nxt, Q, &mbq);
        double2* slot = a.slot + (long long)(cur.plane % 3) * slot_e;
#if MXB_PIPE_DISCARD
        if (cur.kind == U_C) {
            char* row = reinterpret_cast<char*>(slot + (long long)cur.idx * L * 3);
            for (int j = threadIdx.x; j < 3 * L * 16 / 128; j += 96)
                asm volatile("discard.global.L2 [%0], 128;" ::"l"(row + (size_t)j * 128) : "memory");
        }
#endif
        bool inverse = cur.kind == U_C;
        if (cur.kind != U_C) {
            fw::fft1024<-1, MXB_HALF_IN != 0>(v, Wc, lane, tw);
            if (cur.kind == U_A) {
                // ---- y forward of row z = idx -> slot row [ky][c]: one bulk store
                __syncthreads();
#pragma unroll
                for (int k = 0; k < 32; ++k) W[(lane + 32 * k) * 3 + c] = v[fw::p32(k)];
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncthreads();
                if (threadIdx.x == 0) bulk_store(slot + (long long)cur.idx * L * 3, 3 * L);
            } else {
                // ---- B: * K between the z transforms of column ky = idx
                const int ky = cur.idx;
                __syncwarp();
#pragma unroll
                for (int k = 0; k < 32; ++k) Wc[lane + 32 * k] = v[fw::p32(k)];
                __syncthreads();
                const bool fy = 2 * ky > L;
                const double s = a.scale;
                const double2* krow = Kp2 + ((long long)cur.plane * L2 + (fy ? L - ky : ky)) * L2 * 3;
                for (int kz = threadIdx.x; kz < L; kz += 96) {
                    const bool fz = 2 * kz > L;
                    const double2* kr = krow + (fz ? L - kz : kz) * 3;
                    const double2 q01 = __ldg(kr), q23 = __ldg(kr + 1), q45 = __ldg(kr + 2);
                    const double kxx = q01.x, kyy = q23.y, kzz = q45.y;
                    const double kxy = fy ? -q01.y : q01.y;
                    const double kxz = fz ? -q23.x : q23.x;
                    const double kyz = (fy != fz) ? -q45.x : q45.x;
                    const double2 m0 = W[kz], m1 = W[L + kz], m2 = W[2 * L + kz];
                    const double2 h0 = make_double2(kxx * m0.x + kxy * m1.x + kxz * m2.x,
                                                    kxx * m0.y + kxy * m1.y + kxz * m2.y);
                    const double2 h1 = make_double2(kxy * m0.x + kyy * m1.x + kyz * m2.x,
                                                    kxy * m0.y + kyy * m1.y + kyz * m2.y);
                    const double2 h2 = make_double2(kxz * m0.x + kyz * m1.x + kzz * m2.x,
                                                    kxz * m0.y + kyz * m1.y + kzz * m2.y);
                    W[kz] = make_double2(h0.x * s, h0.y * s);
                    W[L + kz] = make_double2(h1.x * s, h1.y * s);
                    W[2 * L + kz] = make_double2(h2.x * s, h2.y * s);
                }
                __syncthreads();
#pragma unroll
                for (int m = 0; m < 32; ++m) v[m] = Wc[lane + 32 * m];
                __syncthreads();
                inverse = true;
            }
        }
        if (inverse) {
            fw::fft1024<1>(v, Wc, lane, tw);
            __syncthreads();
#pragma unroll
            for (int k = 0; k < 16; ++k) W[(lane + 32 * k) * 3 + c] = v[fw::p32(k)];
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (threadIdx.x == 0) {
                if (cur.kind == U_C) {
                    // ---- y inverse of row z = idx -> XP row: one bulk store
                    bulk_store(a.XP + xp_row(a, plane_xp, cur.plane, cur.idx, N * 3), 3 * N);
                } else {
                    // ---- B: the column back into the slot as two tensor boxes
                    const int y0 = (cur.plane % 3) * N;
                    tma_store_2d(&tmap_slot, cur.idx * 6, y0, W);
                    tma_store_2d(&tmap_slot, cur.idx * 6, y0 + 256, W + 768);
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                }
            }
        }
        if (threadIdx.x == 0) {
            tk_sh = tk2;
            pending = cur;
        }
        __syncthreads();
        cur = nxt;
        nxt = tmap(tk_sh);
        in_q = staged_next;
    }
    if (threadIdx.x == 0) {
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        asm volatile("fence.proxy.async.global;" ::: "memory");
        if (pending.kind != U_NONE) sc.signal(pending);
    }
}

// ---------------------------------------------------------------------------
// warp-FFT variant, L = 512 (n = 256): two lines per warp (fw::fft512x2), so a
// unit is a pair: A and C take two z rows, B two adjacent ky columns.  The
// scheduler runs on pair units (n/2 A and C units, L/2 B units per plane);
// staging layouts are [line][z or y][c], 48 KB per CTA, four CTAs per SM.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(96, 4)
k_yz_pipe_w512(PipeArgs a, const double2* __restrict__ tw, const int* __restrict__ halt) {
    if (halt && *halt) return;
    constexpr int L = 512, N = 256, L2 = L / 2 + 1, NU = N / 2, LU = L / 2;
    extern __shared__ double2 W[];                 // 3 x 1024
    __shared__ long long next_ticket;
    __shared__ int flag;
    __shared__ alignas(8) unsigned long long mbar;  // bulk row copies (A, C)
    const int hx = a.hx;
    const long long plane_xp = (long long)a.nzl * N * 3, slot_e = (long long)N * L * 3;
    const int c = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double2* Wc = W + c * 1024;
    PipeArgs au = a;
    au.n = NU;
    const Sched sc(au, LU, halt);
    const TicketMap tmap{hx, NU, LU};
    const double2* __restrict__ Kp2 = reinterpret_cast<const double2*>(a.Kp);

    auto stage = [&](const Unit& u) {
        double2* slot = a.slot + (long long)(u.plane % 3) * slot_e;
        if (u.kind == U_A) {   // rows 2 idx, 2 idx + 1 of XP: contiguous
            if (threadIdx.x == 0)
                bulk_g2s(W, a.XP + xp_row(a, plane_xp, u.plane, 2 * u.idx, N * 3), 2 * N * 3 * 16, &mbar);
        } else if (u.kind == U_B) {   // columns 2 idx, 2 idx + 1: 96 contiguous bytes per z
            const int ky0 = 2 * u.idx;
            for (int j = threadIdx.x; j < 6 * N; j += 96) {
                const int z = j / 6, r = j - 6 * z, ln = r / 3, cc = r - 3 * ln;
                cp_async16(&W[(ln * N + z) * 3 + cc], slot + ((long long)z * L + ky0 + ln) * 3 + cc, true);
            }
            if (threadIdx.x < 2) {
                const int ky = ky0 + threadIdx.x, kyq = 2 * ky > L ? L - ky : ky;
                if (a.cplx) {
                    const double* kr = a.Kp + ((long long)u.plane * L + ky) * L * 12;
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(kr), "r"(L * 96) : "memory");
                } else {
                    const double* kr = a.Kp + ((long long)u.plane * L2 + kyq) * L2 * 6;
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(kr), "r"(L2 * 48) : "memory");
                }
            }
        } else {   // slot rows 2 idx, 2 idx + 1: contiguous
            if (threadIdx.x == 0) bulk_g2s(W, slot + (long long)(2 * u.idx) * L * 3, 2 * L * 3 * 16, &mbar);
        }
        cp_async_commit();
    };
    unsigned mphase = 0;

    if (threadIdx.x == 0) {
        next_ticket = atomicAdd(sc.ticket(), 1u);
        mbar_init(&mbar);
    }
    __syncthreads();
    Unit cur = tmap(next_ticket);
    Unit pending{U_NONE, 0, 0};

    while (cur.kind != U_NONE) {
        if (!sc.wait_ready(cur, &flag, pending)) return;
        stage(cur);
        cp_async_wait_all();
        if (cur.kind != U_B) {
            mbar_wait(&mbar, mphase);
            mphase ^= 1u;
        }
        if (pending.kind != U_NONE) {
            sc.signal(pending);
            pending.kind = U_NONE;
        }
        __syncthreads();
        double2* slot = a.slot + (long long)(cur.plane % 3) * slot_e;
#if MXB_PIPE_DISCARD
        if (cur.kind == U_C) {
            char* rows = reinterpret_cast<char*>(slot + (long long)(2 * cur.idx) * L * 3);
            for (int j = threadIdx.x; j < 2 * L * 3 * 16 / 128; j += 96)
                asm volatile("discard.global.L2 [%0], 128;" ::"l"(rows + (size_t)j * 128) : "memory");
        }
#endif
        double2 xa[16], xb[16], v[32];
        if (cur.kind == U_C) {
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                xa[m] = W[(lane + 32 * m) * 3 + c];
                xb[m] = W[(L + lane + 32 * m) * 3 + c];
            }
        } else {
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                xa[m] = m < 8 ? W[(lane + 32 * m) * 3 + c] : make_double2(0.0, 0.0);
                xb[m] = m < 8 ? W[(N + lane + 32 * m) * 3 + c] : make_double2(0.0, 0.0);
            }
        }
        __syncthreads();   // W becomes the transpose tiles
        const int line = lane >> 4, k1 = lane & 15;
        bool inverse = cur.kind == U_C;
        if (cur.kind != U_C) {
            fw::fft512x2<-1>(xa, xb, v, Wc, lane, tw);
            if (threadIdx.x == 0) next_ticket = atomicAdd(sc.ticket(), 1u);
            __syncthreads();
            if (cur.kind == U_A) {
                // ---- y forward of rows 2 idx (+1) -> slot rows [ky][c]
#pragma unroll
                for (int k2 = 0; k2 < 32; ++k2) W[(line * L + k1 + 16 * k2) * 3 + c] = v[fw::p32(k2)];
                __syncthreads();
                double2* dst = slot + (long long)(2 * cur.idx) * L * 3;
                for (int j = threadIdx.x; j < 2 * L * 3; j += 96) st_l2(dst + j, W[j]);
            } else {
                // ---- B: * K between the z transforms of columns 2 idx (+1)
                const int ky0 = 2 * cur.idx;
#pragma unroll
                for (int k2 = 0; k2 < 32; ++k2) W[c * 1024 + line * L + k1 + 16 * k2] = v[fw::p32(k2)];
                __syncthreads();
                const double s = a.scale;
                if (a.cplx) {
                    for (int t = threadIdx.x; t < 2 * L; t += 96) {
                        const int ln = t / L, kz = t - ln * L;
                        kmul_complex(Kp2 + (((long long)cur.plane * L + ky0 + ln) * L + kz) * 6, W[t], W[1024 + t],
                                     W[2048 + t], s);
                    }
                }
#if MXB_PIPE_KPAIR_512
                // kz and L - kz share a parity-reduced entry: one load, two updates
                for (int t = a.cplx ? 2 * L2 : threadIdx.x; t < 2 * L2; t += 96) {
                    const int ln = t / L2, q = t - ln * L2, ky = ky0 + ln;
                    const bool fy = 2 * ky > L;
                    const double2* kr = Kp2 + (((long long)cur.plane * L2 + (fy ? L - ky : ky)) * L2 + q) * 3;
                    const double2 q01 = __ldg(kr), q23 = __ldg(kr + 1), q45 = __ldg(kr + 2);
                    const double kxx = q01.x, kyy = q23.y, kzz = q45.y;
                    const double kxy = fy ? -q01.y : q01.y;
                    const double kyz0 = fy ? -q45.x : q45.x;
                    auto apply = [&](int e, double kxz, double kyz) {
                        const double2 m0 = W[e], m1 = W[1024 + e], m2 = W[2048 + e];
                        const double2 h0 = make_double2(kxx * m0.x + kxy * m1.x + kxz * m2.x,
                                                        kxx * m0.y + kxy * m1.y + kxz * m2.y);
                        const double2 h1 = make_double2(kxy * m0.x + kyy * m1.x + kyz * m2.x,
                                                        kxy * m0.y + kyy * m1.y + kyz * m2.y);
                        const double2 h2 = make_double2(kxz * m0.x + kyz * m1.x + kzz * m2.x,
                                                        kxz * m0.y + kyz * m1.y + kzz * m2.y);
                        W[e] = make_double2(h0.x * s, h0.y * s);
                        W[1024 + e] = make_double2(h1.x * s, h1.y * s);
                        W[2048 + e] = make_double2(h2.x * s, h2.y * s);
                    };
                    apply(ln * L + q, q23.x, kyz0);
                    if (q != 0 && q != L / 2) apply(ln * L + L - q, -q23.x, -kyz0);
                }
#else
                for (int t = a.cplx ? 2 * L : threadIdx.x; t < 2 * L; t += 96) {
                    const int ln = t / L, kz = t - ln * L, ky = ky0 + ln;
                    const bool fy = 2 * ky > L, fz = 2 * kz > L;
                    const double2* kr = Kp2 + (((long long)cur.plane * L2 + (fy ? L - ky : ky)) * L2 +
                                               (fz ? L - kz : kz)) * 3;
                    const double2 q01 = __ldg(kr), q23 = __ldg(kr + 1), q45 = __ldg(kr + 2);
                    const double kxx = q01.x, kyy = q23.y, kzz = q45.y;
                    const double kxy = fy ? -q01.y : q01.y;
                    const double kxz = fz ? -q23.x : q23.x;
                    const double kyz = (fy != fz) ? -q45.x : q45.x;
                    const double2 m0 = W[t], m1 = W[1024 + t], m2 = W[2048 + t];
                    const double2 h0 = make_double2(kxx * m0.x + kxy * m1.x + kxz * m2.x,
                                                    kxx * m0.y + kxy * m1.y + kxz * m2.y);
                    const double2 h1 = make_double2(kxy * m0.x + kyy * m1.x + kyz * m2.x,
                                                    kxy * m0.y + kyy * m1.y + kyz * m2.y);
                    const double2 h2 = make_double2(kxz * m0.x + kyz * m1.x + kzz * m2.x,
                                                    kxz * m0.y + kyz * m1.y + kzz * m2.y);
                    W[t] = make_double2(h0.x * s, h0.y * s);
                    W[1024 + t] = make_double2(h1.x * s, h1.y * s);
                    W[2048 + t] = make_double2(h2.x * s, h2.y * s);
                }
#endif
                __syncthreads();
#pragma unroll
                for (int m = 0; m < 16; ++m) {
                    xa[m] = Wc[lane + 32 * m];
                    xb[m] = Wc[L + lane + 32 * m];
                }
                __syncthreads();   // tiles reused by the inverse
                inverse = true;
            }
        }
        if (inverse) {
            fw::fft512x2<1>(xa, xb, v, Wc, lane, tw);
            if (cur.kind == U_C && threadIdx.x == 0) next_ticket = atomicAdd(sc.ticket(), 1u);
            __syncthreads();
#pragma unroll
            for (int k2 = 0; k2 < 16; ++k2) W[(line * N + k1 + 16 * k2) * 3 + c] = v[fw::p32(k2)];   // n < N kept
            __syncthreads();
            if (cur.kind == U_C) {
                // ---- y inverse of rows 2 idx (+1) -> XP rows (contiguous)
                double2* dst = a.XP + xp_row(a, plane_xp, cur.plane, 2 * cur.idx, N * 3);
                for (int j = threadIdx.x; j < 2 * N * 3; j += 96) st_stream(dst + j, W[j]);
            } else {
                // ---- B: columns back into the slot (96 contiguous bytes per z)
                const int ky0 = 2 * cur.idx;
                for (int j = threadIdx.x; j < 6 * N; j += 96) {
                    const int z = j / 6, r = j - 6 * z, ln = r / 3, cc = r - 3 * ln;
                    st_l2(slot + ((long long)z * L + ky0 + ln) * 3 + cc, W[(ln * N + z) * 3 + cc]);
                }
            }
        }
        __syncthreads();
        pending = cur;
        cur = tmap(next_ticket);
    }
    if (pending.kind != U_NONE) sc.signal(pending);
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static int sm_count() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}

template <int L>
static int pipe_launch_L(const PipeArgs& a, const double2* tw, cudaStream_t st, const int* halt) {
    constexpr int T = PipeCfg<L>::T;
    const size_t smem = (size_t)(PipeCfg<L>::XE + PipeCfg<L>::SE) * sizeof(double2);
    static int grid = 0;
    if (!grid) {
        MXB_CUDA(cudaFuncSetAttribute(k_yz_pipe<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        MXB_CUDA(cudaFuncSetAttribute(k_yz_pipe<L>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        int per_sm = 0;
        MXB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_yz_pipe<L>, T, smem));
        if (per_sm < 1) { set_error("pipeline kernel does not fit on an SM"); return MXB_EINVAL; }
        grid = per_sm * sm_count();
        if (getenv("MXB_PIPE_VERBOSE")) {
            cudaFuncAttributes fa;
            cudaFuncGetAttributes(&fa, k_yz_pipe<L>);
            fprintf(stderr, "k_yz_pipe<%d>: regs %d smem %zu per_sm %d grid %d\n", L, fa.numRegs, smem,
                    per_sm, grid);
        }
    }
    int g = grid;
    if (const char* e = getenv("MXB_PIPE_GRID")) g = atoi(e) > 0 ? atoi(e) : g;
    MXB_CUDA(cudaMemsetAsync(a.sync, 0, (2 + 2 * (size_t)a.hx + 3 * (size_t)a.n) * sizeof(unsigned), st));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)g);
    cfg.blockDim = dim3((unsigned)T);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    MXB_CUDA(cudaLaunchKernelEx(&cfg, k_yz_pipe<L>, a, tw, halt));
    return MXB_OK;
}

// shapes the pipeline covers: 3-D, ny == nz, power-of-two padded length L <= 1024
bool pipe_shape_ok(int ny, int nz) {
    const int L = 2 * ny;
    return ny == nz && ny >= 8 && L <= 1024 && (L & (L - 1)) == 0;
}

static int pipe_launch_warp512(const PipeArgs& a, const double2* tw, cudaStream_t st, const int* halt) {
    const size_t smem = (size_t)(3 * 1024) * sizeof(double2);
    static int grid = 0;
    if (!grid) {
        MXB_CUDA(cudaFuncSetAttribute(k_yz_pipe_w512, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        MXB_CUDA(cudaFuncSetAttribute(k_yz_pipe_w512, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        int per_sm = 0;
        MXB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_yz_pipe_w512, 96, smem));
        if (per_sm < 1) { set_error("pipeline kernel does not fit on an SM"); return MXB_EINVAL; }
        grid = per_sm * sm_count();
        if (getenv("MXB_PIPE_VERBOSE")) {
            cudaFuncAttributes fa;
            cudaFuncGetAttributes(&fa, k_yz_pipe_w512);
            fprintf(stderr, "k_yz_pipe_w512: regs %d smem %zu per_sm %d grid %d\n", fa.numRegs, smem, per_sm, grid);
        }
    }
    int g = grid;
    if (const char* e = getenv("MXB_PIPE_GRID")) g = atoi(e) > 0 ? atoi(e) : g;
    MXB_CUDA(cudaMemsetAsync(a.sync, 0, (2 + 2 * (size_t)a.hx + 3 * (size_t)a.n) * sizeof(unsigned), st));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)g);
    cfg.blockDim = dim3(96u);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    MXB_CUDA(cudaLaunchKernelEx(&cfg, k_yz_pipe_w512, a, tw, halt));
    return MXB_OK;
}

// the slot ring as a 2-D float64 tensor: rows (slot, z), L * 6 values each;
// box {6, 256} = one ky column over 256 z
static int make_slot_map(CUtensorMap* tm, void* slot, int L, int n) {
    return make_map_2d_f64(tm, slot, (unsigned long long)L * 6, 3ULL * n, (unsigned long long)L * 6 * sizeof(double),
                           6, 256);
}

static int pipe_launch_warpq(const PipeArgs& a, const double2* tw, cudaStream_t st, const int* halt) {
    const size_t smem = (size_t)(3 * 1024 + 3 * 512) * sizeof(double2);
    static int grid = 0;
    if (!grid) {
        MXB_CUDA(cudaFuncSetAttribute(k_yz_pipe_wq, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        MXB_CUDA(cudaFuncSetAttribute(k_yz_pipe_wq, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        int per_sm = 0;
        MXB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_yz_pipe_wq, 96, smem));
        if (per_sm < 1) { set_error("pipeline kernel does not fit on an SM"); return MXB_EINVAL; }
        grid = per_sm * sm_count();
        if (getenv("MXB_PIPE_VERBOSE")) fprintf(stderr, "k_yz_pipe_wq: per_sm %d grid %d\n", per_sm, grid);
    }
    MXB_CUDA(cudaMemsetAsync(a.sync, 0, (2 + 2 * (size_t)a.hx + 3 * (size_t)a.n) * sizeof(unsigned), st));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(96u);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CUtensorMap tm;
    if (make_slot_map(&tm, a.slot, 1024, a.n)) return MXB_ECUDA;
    MXB_CUDA(cudaLaunchKernelEx(&cfg, k_yz_pipe_wq, a, tw, halt, tm));
    return MXB_OK;
}

static int pipe_launch_warp(const PipeArgs& a, const double2* tw, cudaStream_t st, const int* halt) {
    const size_t smem = (size_t)(3 * 1024) * sizeof(double2);
    static int grid = 0;
    if (!grid) {
        MXB_CUDA(cudaFuncSetAttribute(k_yz_pipe_w, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        MXB_CUDA(cudaFuncSetAttribute(k_yz_pipe_w, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        int per_sm = 0;
        MXB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_yz_pipe_w, 96, smem));
        if (per_sm < 1) { set_error("pipeline kernel does not fit on an SM"); return MXB_EINVAL; }
        grid = per_sm * sm_count();
        if (getenv("MXB_PIPE_VERBOSE")) {
            cudaFuncAttributes fa;
            cudaFuncGetAttributes(&fa, k_yz_pipe_w);
            fprintf(stderr, "k_yz_pipe_w: regs %d smem %zu per_sm %d grid %d\n", fa.numRegs, smem, per_sm, grid);
        }
    }
    int g = grid;
    if (const char* e = getenv("MXB_PIPE_GRID")) g = atoi(e) > 0 ? atoi(e) : g;
    MXB_CUDA(cudaMemsetAsync(a.sync, 0, (2 + 2 * (size_t)a.hx + 3 * (size_t)a.n) * sizeof(unsigned), st));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)g);
    cfg.blockDim = dim3(96u);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CUtensorMap tm;
    if (make_slot_map(&tm, a.slot, 1024, a.n)) return MXB_ECUDA;
    MXB_CUDA(cudaLaunchKernelEx(&cfg, k_yz_pipe_w, a, tw, halt, tm));
    return MXB_OK;
}

// the complex-spectra pipeline (the reference's tensor, from_packed) exists for
// the warp-FFT kernels only
bool pipe_cplx_ok(int L) {
    const char* we = getenv("MXB_PIPE_WARP");
    const char* pe = getenv("MXB_PIPE_PREFETCH");
    if ((we && we[0] == '0') || (pe && pe[0] == '1')) return false;
    return L == 512 || L == 1024;
}

int pipe_yz(double2* XP, double2* slot, const double* Kp, unsigned* bar, int hx, int n, double scale,
            const double2* tw, cudaStream_t st, const int* halt, int cplx, int nzl, long long gstride) {
    const int nzl_ = nzl > 0 ? nzl : n;
    const PipeArgs a{XP, slot, Kp, bar, hx, n, scale, cplx, nzl_, nzl_ != n ? gstride / nzl_ : 0};
    if (a.nzl != n && (a.nzl < 2 || (a.nzl & (a.nzl - 1)) || n % a.nzl || gstride % a.nzl)) {
        set_error("pipeline slab: the local planes must be a power of two dividing n");
        return MXB_EINVAL;
    }
    if (cplx && !pipe_cplx_ok(2 * n)) { set_error("complex-spectra pipeline needs the warp kernels (L = 512 / 1024)"); return MXB_EINVAL; }
    // warp-FFT variant by default at L = 1024 (27.6 vs 32.1 ms per evaluation at
    // 512^3; within 4e-16 of the 5-pass path).  MXB_PIPE_WARP=0 selects the
    // radix-16 pipeline, which is bit-identical to the 5-pass path.
    const char* we = getenv("MXB_PIPE_WARP");
    const bool warp = !(we && we[0] == '0');
    if (2 * n == 1024 && warp) {
        const char* pe = getenv("MXB_PIPE_PREFETCH");
        if (pe && pe[0] == '1') return pipe_launch_warpq(a, tw, st, halt);
        return pipe_launch_warp(a, tw, st, halt);
    }
    if (2 * n == 512 && warp) return pipe_launch_warp512(a, tw, st, halt);
    switch (2 * n) {
        case 16: return pipe_launch_L<16>(a, tw, st, halt);
        case 32: return pipe_launch_L<32>(a, tw, st, halt);
        case 64: return pipe_launch_L<64>(a, tw, st, halt);
        case 128: return pipe_launch_L<128>(a, tw, st, halt);
        case 256: return pipe_launch_L<256>(a, tw, st, halt);
        case 512: return pipe_launch_L<512>(a, tw, st, halt);
        case 1024: return pipe_launch_L<1024>(a, tw, st, halt);
        default: set_error("no pipeline kernel for this shape"); return MXB_EINVAL;
    }
}

// K (complex full spectra [kz][ky][hxp][6], exactly real) -> Kp[kx][ky'][kz'][6]
__global__ void k_planes_quarter(const double2* __restrict__ K, double* __restrict__ Kp, int L, int hx,
                                 int hxp, int kx0) {
    const int L2 = L / 2 + 1;
    const long long tot = (long long)hx * L2 * L2 * 6;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
         i += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(i % 6);
        long long r = i / 6;
        const int kz = (int)(r % L2);
        r /= L2;
        const int ky = (int)(r % L2);
        const int kx = (int)(r / L2);
        Kp[i] = K[(((long long)kz * L + ky) * hxp + kx0 + kx) * 6 + c].x;
    }
}

int pipe_quarter(const double2* K, double* Kp, int L, int hx, int hxp, cudaStream_t st, int kx0) {
    k_planes_quarter<<<148 * 8, 256, 0, st>>>(K, Kp, L, hx, hxp, kx0);
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

}  // namespace mxb

namespace mxb {

// K (complex full spectra [kz][ky][hxp][6]) -> Kx[kx][ky][kz][6] complex, the
// B units' kernel rows contiguous (L x 96 B per (kx, ky))
__global__ void k_planes_complex(const double2* __restrict__ K, double2* __restrict__ Kx, int L, int hx, int hxp,
                                 int kx0) {
    const long long tot = (long long)hx * L * L * 6;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
         i += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(i % 6);
        long long r = i / 6;
        const int kz = (int)(r % L);
        r /= L;
        const int ky = (int)(r % L);
        const int kx = (int)(r / L);
        Kx[i] = K[(((long long)kz * L + ky) * hxp + kx0 + kx) * 6 + c];
    }
}

int pipe_complex(const double2* K, double2* Kx, int L, int hx, int hxp, cudaStream_t st, int kx0) {
    k_planes_complex<<<148 * 8, 256, 0, st>>>(K, Kx, L, hx, hxp, kx0);
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

}  // namespace mxb
