// L2-resident y/z pipeline over kx planes (single GPU, 3-D, symmetric kernel).
//
// The 5-pass demag evaluation moves every intermediate through HBM; at 512^3
// the y/z middle (y forward, z fused, y inverse) alone is ~79 GB per
// evaluation.  Here one persistent cooperative kernel walks the hx kx-planes
// in ticks.  In tick t it runs, spread over all CTAs,
//   A  y forward of plane t      : XP rows (HBM) -> slot[t % 3]   [z][ky][c]
//   B  z fwd * K * z inv, plane t-1 : in place in slot[(t-1) % 3]
//   C  y inverse of plane t-2    : slot[(t-2) % 3] -> XP rows (HBM)
// and a grid barrier separates ticks.  The three slots (3 * nz * py * 48 B,
// 75 MB at 512^3) stay in L2, so HBM only sees XP once each way plus the
// kernel spectra: ~19 GB per evaluation at 512^3.
//
// Layouts: XP[kx][z][y][c] (plane-major x-pass output, written by
// k_r2c_fast with CH = CHP = 1), Kp[kx][ky'][kz'][6] real quarter spectra
// with ky' = min(ky, py-ky), kz' = min(kz, pz-kz) and the parity signs of
// XY/XZ/YZ (as k_quarterize).  The transforms are the same register-resident
// radix-16 Stockham code (fft_fast.cuh) with the same twiddles as the 5-pass
// kernels, so both paths produce identical results.
//
// Every unit is one line triple (the 3 components): 3 * L/16 threads, two
// CTAs per SM.  HBM-sourced inputs (XP rows for A, K rows for B) are
// prefetched with cp.async into a staging buffer while the previous unit
// computes; slot traffic (L2) is loaded and stored cooperatively through
// shared memory so every warp access is contiguous.
#include <stdio.h>
#include <stdlib.h>

#include "demag.cuh"
#include "fft_fast.cuh"

namespace mxb {

using namespace ff;

struct PipeArgs {
    double2* XP;          // [hx][nz][ny][3], input and output (in place)
    double2* slot;        // 3 x [nz][L][3]
    const double* Kp;     // [hx][L/2+1][L/2+1][6]
    unsigned* sync;       // [ticket, abort, doneA[hx], doneB[hx], doneC[hx]], zeroed per launch
    int hx, n;            // planes; non-zero rows ny == nz == n
    double scale;
};

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

// Tickets are handed out in rounds r = 0 .. hx+1; round r holds, in order,
//   A(r) [n units, r < hx], C(r-2) [n units, 2 <= r], B(r-1) [L units, 1 <= r <= hx].
// Every dependency (B(p) <- A(p), C(p) <- B(p), A(p) <- C(p-3) for the slot
// reuse) then lies in the previous round at least n tickets back, so with
// n >= the number of CTAs a unit almost never waits.
__device__ __forceinline__ int ky_of(int q, int L) {
    // pair ky with L - ky on neighbouring tickets: the shared K row is read once from HBM
    return q == 0 ? 0 : ((q & 1) ? (q + 1) / 2 : L - q / 2);
}

// ticket -> unit (hx >= 2): round 0 = A(0); round 1 = A(1), B(0);
// rounds 2..hx-1 = A(r), C(r-2), B(r-1); round hx = C(hx-2), B(hx-1); round hx+1 = C(hx-1)
__device__ __forceinline__ Unit decode(long long k, int hx, int n, int L) {
    if (k < n) return {U_A, 0, (int)k};
    k -= n;
    if (k < n) return {U_A, 1, (int)k};
    k -= n;
    if (k < L) return {U_B, 0, ky_of((int)k, L)};
    k -= L;
    const long long full = 2LL * n + L, nfull = hx - 2;
    if (k < nfull * full) {
        const int r = 2 + (int)(k / full);
        int o = (int)(k % full);
        if (o < n) return {U_A, r, o};
        o -= n;
        if (o < n) return {U_C, r - 2, o};
        return {U_B, r - 1, ky_of(o - n, L)};
    }
    k -= nfull * full;
    if (k < n) return {U_C, hx - 2, (int)k};
    k -= n;
    if (k < L) return {U_B, hx - 1, ky_of((int)k, L)};
    k -= L;
    if (k < n) return {U_C, hx - 1, (int)k};
    return {U_NONE, 0, 0};
}

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
    __shared__ long long next_ticket;
    __shared__ int flag;
    double2* X = sm;
    double2* S = sm + PipeCfg<L>::XE;
    const int n = a.n, hx = a.hx;
    const long long plane_xp = (long long)n * n * 3;       // XP elements per kx plane
    const long long slot_e = (long long)n * L * 3;         // slot elements
    const int b = threadIdx.x / TPL, t = threadIdx.x - (threadIdx.x / TPL) * TPL;
    unsigned* ticket = a.sync;
    unsigned* abort_w = a.sync + 1;
    unsigned* doneA = a.sync + 2;
    unsigned* doneB = doneA + hx;
    unsigned* doneC = doneB + hx;

    // counter a unit waits on, and its target
    auto dep = [&](const Unit& u, const unsigned** c, unsigned* target) {
        if (u.kind == U_A) {
            if (u.plane < 3) return false;
            *c = doneC + (u.plane - 3);
            *target = (unsigned)n;
        } else if (u.kind == U_B) {
            *c = doneA + u.plane;
            *target = (unsigned)n;
        } else {
            *c = doneB + u.plane;
            *target = (unsigned)L;
        }
        return true;
    };
    auto ready = [&](const Unit& u) {   // thread 0
        const unsigned* c;
        unsigned tg;
        return !dep(u, &c, &tg) || ld_acquire(c) >= tg;
    };
    // thread 0 waits (2 s cap, then every CTA leaves: results are then garbage
    // but the device stays usable); returns false on abort
    auto wait_ready = [&](const Unit& u) {
        if (threadIdx.x == 0) {
            flag = 1;
            const unsigned* c;
            unsigned tg;
            if (dep(u, &c, &tg)) {
                const unsigned long long t0 = gtimer();
                while (ld_acquire(c) < tg) {
                    __nanosleep(32);
                    if (ld_acquire(abort_w)) { flag = 0; break; }
                    if (gtimer() - t0 > 2000000000ull) {
                        printf("k_yz_pipe: wait timeout cta %d kind %d plane %d have %u need %u\n", blockIdx.x,
                               u.kind, u.plane, ld_acquire(c), tg);
                        atomicExch(abort_w, 1u);
                        flag = 0;
                        break;
                    }
                }
            }
        }
        __syncthreads();
        return flag != 0;
    };
    auto signal = [&](const Unit& u) {   // after a __syncthreads that follows the unit's stores
        if (threadIdx.x == 0) {
            __threadfence();
            unsigned* c = u.kind == U_A ? doneA : (u.kind == U_B ? doneB : doneC);
            atomicAdd(c + u.plane, 1u);
        }
    };

    // unit inputs, staged in S with cp.async: A an XP row (HBM), B a slot
    // column (L2), C a slot row (L2); B also stages its K rows (HBM) over its
    // own forward FFT
    auto stage_in = [&](const Unit& u) {
        if (u.kind == U_A) {
            const double2* src = a.XP + u.plane * plane_xp + (long long)u.idx * n * 3;
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

    if (threadIdx.x == 0) next_ticket = atomicAdd(ticket, 1u);
    __syncthreads();
    Unit cur = decode(next_ticket, hx, n, L);
    bool staged = false;

    while (cur.kind != U_NONE) {
        if (!staged) {
            if (!wait_ready(cur)) return;
            stage_in(cur);
        }
        __syncthreads();   // next_ticket / flag are free
        if (threadIdx.x == 0) next_ticket = atomicAdd(ticket, 1u);
        double2* slot = a.slot + (long long)(cur.plane % 3) * slot_e;
        const int nin = cur.kind == U_C ? L : n;
        double2 v[R];
        cp_async_wait_all();
        __syncthreads();
        const Unit nxt = decode(next_ticket, hx, n, L);
        if (threadIdx.x == 0) flag = nxt.kind != U_NONE && ready(nxt);
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
            double2* dst = a.XP + cur.plane * plane_xp + (long long)cur.idx * n * 3;
            for (int j = threadIdx.x; j < 3 * n; j += T) st_stream(dst + j, X[j]);
        }
        __syncthreads();
        signal(cur);
        cur = nxt;
        staged = staged_next;
    }
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
    MXB_CUDA(cudaMemsetAsync(a.sync, 0, (2 + 3 * (size_t)a.hx) * sizeof(unsigned), st));
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

int pipe_yz(double2* XP, double2* slot, const double* Kp, unsigned* bar, int hx, int n, double scale,
            const double2* tw, cudaStream_t st, const int* halt) {
    const PipeArgs a{XP, slot, Kp, bar, hx, n, scale};
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
                                 int hxp) {
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
        Kp[i] = K[(((long long)kz * L + ky) * hxp + kx) * 6 + c].x;
    }
}

int pipe_quarter(const double2* K, double* Kp, int L, int hx, int hxp, cudaStream_t st) {
    k_planes_quarter<<<148 * 8, 256, 0, st>>>(K, Kp, L, hx, hxp);
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

}  // namespace mxb
