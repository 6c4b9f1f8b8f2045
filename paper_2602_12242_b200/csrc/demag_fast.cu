// Fast-path kernels of the demag pipeline for power-of-two padded lengths:
// register-resident radix-16 Stockham FFTs (fft_fast.cuh) in persistent
// CTAs that stage the NEXT tile's inputs with cp.async while the current
// tile is transformed, so HBM traffic overlaps the FFT arithmetic.
//
//   x rows  : real r2c / c2r of length px through one complex FFT of px/2
//   columns : strided c2c lines (y passes), lines fastest in shared memory
//   fused   : forward c2c * 3x3 kernel multiply * inverse c2c along z (or y
//             for films); the kernel rows of the tile are staged in shared
//             memory too, in parity-reduced (quarter) or complex storage.
// Same buffer layouts as the generic kernels in demag.cu.
#include <stdlib.h>

#include <map>
#include <mutex>
#include <set>
#include <utility>

#include "demag.cuh"
#include "fft_fast.cuh"

namespace mxb {

using namespace ff;

template <int L, int RMAX = 16> struct Cfg {
    static constexpr int R = L >= RMAX ? RMAX : (L < 1 ? 1 : L);
    static constexpr int TPL = L / R;
    // columns: ~256 threads, at least 2 lines (32-byte segments)
    static constexpr int NLc = (256 * R / L) >= 2 ? (256 * R / L) : 2;
    // fused: NK kx columns x 3 components
    static constexpr int NKraw = 256 * R / (3 * L);
    static constexpr int NKf = NKraw < 2 ? 2 : (NKraw > 8 ? 8 : NKraw);   // >= 2: 96-byte aligned chunks
    // rows (M = L complex points per row): NR rows x 3 components
    static constexpr int NRr = (256 * R / (3 * L)) >= 1 ? (256 * R / (3 * L)) : 1;
};

// ---------------------------------------------------------------------------
// strided columns (y passes)
// ---------------------------------------------------------------------------
struct ColArgs {
    const double2* in;
    double2* out;
    int n_in, n_out;
    long long ES_in, ES_out;
    int Q;
    long long nlines, OS_in, OS_out;
};

template <int L, int DIR, int RM, int NLD>
__global__ void __launch_bounds__(Cfg<L, RM>::NLc / NLD * Cfg<L, RM>::TPL, 2)
k_col_fast(ColArgs a, const double2* __restrict__ tw, const int* __restrict__ halt) {
    if (halt && *halt) return;
    constexpr int R = Cfg<L, RM>::R, TPL = Cfg<L, RM>::TPL, NL = Cfg<L, RM>::NLc / NLD;
    extern __shared__ double2 sm[];
    double2* X = sm;
    double2* S = sm + smem_elems<L, R, NL>();
    const long long ntiles = (a.nlines + NL - 1) / NL;
    const int T = blockDim.x;
    auto prefetch = [&](long long tile) {
        for (int u = threadIdx.x; u < NL * a.n_in; u += T) {
            const int bb = u % NL, e = u / NL;
            const long long g = tile * NL + bb;
            const bool ok = g < a.nlines;
            const long long o = ok ? g / a.Q : 0, q = ok ? g - o * a.Q : 0;
            cp_async16(&S[u], a.in + o * a.OS_in + q + e * a.ES_in, ok);
        }
        cp_async_commit();
    };
    long long tile = blockIdx.x;
    if (tile < ntiles) prefetch(tile);
    const int b = threadIdx.x % NL, t = threadIdx.x / NL;
    for (; tile < ntiles; tile += gridDim.x) {
        cp_async_wait_all();
        __syncthreads();
        double2 v[R];
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const int e = t + m * TPL;
            v[m] = e < a.n_in ? S[e * NL + b] : make_double2(0.0, 0.0);
        }
        __syncthreads();
        const long long nxt = tile + gridDim.x;
        if (nxt < ntiles) prefetch(nxt);
        fft_core<L, R, NL, true, DIR>(v, X, b, t, tw);
        const long long g = tile * NL + b;
        if (g < a.nlines) {
            const long long o = g / a.Q, q = g - o * a.Q;
            double2* dst = a.out + o * a.OS_out + q;
#pragma unroll
            for (int i = 0; i < R; ++i) {
                const int e = out_elem<L, R>(t, i);
                if (e < a.n_out) dst[e * a.ES_out] = v[i];
            }
        }
    }
}

// direct-load variant (no staging): used when the staged input would not
// leave room for two CTAs per SM (e.g. the inverse y pass, n_in = L)
template <int L, int DIR, int RM>
__global__ void __launch_bounds__(Cfg<L, RM>::NLc * Cfg<L, RM>::TPL, 2)
k_col_direct(ColArgs a, const double2* __restrict__ tw, const int* __restrict__ halt) {
    if (halt && *halt) return;
    constexpr int R = Cfg<L, RM>::R, TPL = Cfg<L, RM>::TPL, NL = Cfg<L, RM>::NLc;
    extern __shared__ double2 sm[];
    const int b = threadIdx.x % NL, t = threadIdx.x / NL;
    const long long g = (long long)blockIdx.x * NL + b;
    const bool ok = g < a.nlines;
    const long long o = ok ? g / a.Q : 0, q = ok ? g - o * a.Q : 0;
    const double2* src = a.in + o * a.OS_in + q;
    double2 v[R];
#pragma unroll
    for (int m = 0; m < R; ++m) {
        const int e = t + m * TPL;
        v[m] = (ok && e < a.n_in) ? src[e * a.ES_in] : make_double2(0.0, 0.0);
    }
    fft_core<L, R, NL, true, DIR>(v, sm, b, t, tw);
    double2* dst = a.out + o * a.OS_out + q;
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const int e = out_elem<L, R>(t, i);
        if (ok && e < a.n_out) dst[e * a.ES_out] = v[i];
    }
}

// ---------------------------------------------------------------------------
// CTAs per SM the fused kernels are compiled for: two for the real folded
// kernel modes up to L = 256 (one CTA at 234-244 registers left the SM at 6
// warps: long-y z pass at L = 128 38.0 -> 28.0 ms, 5-pass z at L = 128
// 0.567 -> 0.414 ms, L = 256 -1.6%); one above (L = 1024 would spill 736 B)
template <int L, int KMODE> constexpr int fused_minb() { return (KMODE == 2 || KMODE == 4) && L <= 256 ? 2 : 1; }

// fused forward * multiply * inverse along the outer axis
// K storage: KMODE 0 complex [e*G+g][kx][6]; 2 real quarter [e'][g'][kx][6]
// with e' = min(e, L-e), g' = min(g, G-g) and the parity signs of XY/XZ/YZ;
// 4 (long-y plane-major layout, longy.cu: the contiguous lane is ky, g is kx)
// real [g][ky'][e'][6] with ky' = min(ky, py-ky), py = a.hx.
// Tile order pairs g with G-g so the shared quarter rows are reused from L2.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int g_of(int r, int G) {
    if (r == 0) return 0;
    return (r & 1) ? (r + 1) / 2 : G - r / 2;
}

template <int L, int KMODE, int RM>
__global__ void __launch_bounds__(3 * Cfg<L, RM>::NKf * Cfg<L, RM>::TPL, fused_minb<L, KMODE>())
k_fused_fast(FusedArgs a, const double2* __restrict__ tw, const int* __restrict__ halt) {
    if (halt && *halt) return;
    constexpr int R = Cfg<L, RM>::R, TPL = Cfg<L, RM>::TPL, NK = Cfg<L, RM>::NKf, NL = 3 * NK;
    constexpr bool KQ = KMODE == 2 || KMODE == 4;   // real folded kernel
    constexpr int KROWS = KQ ? (L / 2 + 1) : L;
    constexpr int KCH = KQ ? 3 : 6;   // 16-byte chunks per (row, kx)
    extern __shared__ double2 sm[];
    double2* X = sm;
    double2* S = X + smem_elems<L, R, NL>();
    double2* KS = S + NL * a.n;               // KROWS * NK * KCH chunks
    const int nkt = (a.hx + NK - 1) / NK;
    const long long ntiles = (long long)a.G * nkt;
    const int T = blockDim.x;
    const int G2 = a.G / 2 + 1;
    auto prefetch_x = [&](long long tile) {
        const int r = (int)(tile / nkt), kt = (int)(tile - (long long)r * nkt);
        const int g = g_of(r, a.G), kx0 = kt * NK;
        for (int u = threadIdx.x; u < NL * a.n; u += T) {
            const int bb = u % NL, e = u / NL;
            const int kx = kx0 + bb / 3, c = bb % 3;
            const bool ok = kx < a.hx;
            cp_async16(&S[u], a.X + g * a.GS + (long long)(ok ? kx : 0) * 3 + c + e * a.ES, ok);
        }
        cp_async_commit();
    };
    auto prefetch_k = [&](long long tile) {
        const int r = (int)(tile / nkt), kt = (int)(tile - (long long)r * nkt);
        const int g = g_of(r, a.G), kx0 = kt * NK;
        for (int u = threadIdx.x; u < KROWS * NK * KCH; u += T) {
            const int part = u % KCH, rest = u / KCH;
            const int kl = rest % NK, e = rest / NK;
            const int kx = kx0 + kl;
            const bool ok = kx < a.hx;
            const int kxs = ok ? kx : 0;
            const double2* src;
            if (KMODE == 4) {
                const int ky2 = 2 * kxs > a.hx ? a.hx - kxs : kxs;
                src = reinterpret_cast<const double2*>((const double*)a.K +
                                                       (((long long)g * (a.hx / 2 + 1) + ky2) * KROWS + e) * 6) +
                      part;
            } else if (KMODE == 2) {
                const int g2 = 2 * g > a.G ? a.G - g : g;
                src = reinterpret_cast<const double2*>((const double*)a.K +
                                                       (((long long)e * G2 + g2) * a.hxp + kxs) * 6) + part;
            } else {
                src = (const double2*)a.K + (((long long)e * a.G + g) * a.hxp + kxs) * 6 + part;
            }
            cp_async16(&KS[u], src, ok);
        }
        cp_async_commit();
    };
    long long tile = blockIdx.x;
    if (tile < ntiles) {
        prefetch_x(tile);
        prefetch_k(tile);
    }
    const int b = threadIdx.x % NL, t = threadIdx.x / NL;
    for (; tile < ntiles; tile += gridDim.x) {
        const int r = (int)(tile / nkt), kt = (int)(tile - (long long)r * nkt);
        const int g = g_of(r, a.G), kx0 = kt * NK;
        cp_async_wait_all();
        __syncthreads();
        double2 v[R];
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const int e = t + m * TPL;
            v[m] = e < a.n ? S[e * NL + b] : make_double2(0.0, 0.0);
        }
        __syncthreads();
        const long long nxt = tile + gridDim.x;
        if (nxt < ntiles) prefetch_x(nxt);
        fft_core<L, R, NL, true, -1>(v, X, b, t, tw);
        if (L > R) __syncthreads();
#pragma unroll
        for (int i = 0; i < R; ++i) X[sidx<true, L, R, NL>(b, out_elem<L, R>(t, i))] = v[i];
        __syncthreads();
        // 3x3 symmetric multiply, scaled by 1/(px py pz)
        const bool rg = 2 * g > a.G;
        for (int u = threadIdx.x; u < NK * L; u += T) {
            const int kl = u % NK, e = u / NK;
            if (kx0 + kl >= a.hx) continue;
            const int i0 = sidx<true, L, R, NL>(3 * kl, e);
            const double2 m0 = X[i0], m1 = X[i0 + 1], m2 = X[i0 + 2];
            double2 h0, h1, h2;
            if (KQ) {
                const bool re = 2 * e > L;
                const int e2 = re ? L - e : e;
                const double* k = reinterpret_cast<const double*>(KS + (e2 * NK + kl) * KCH);
                const bool fy = KMODE == 4 ? 2 * (kx0 + kl) > a.hx : (a.e_is_z ? rg : re);
                const bool fz = KMODE == 4 ? re : (a.e_is_z ? re : rg);
                const double kxx = k[0], kyy = k[3], kzz = k[5];
                const double kxy = fy ? -k[1] : k[1];
                const double kxz = fz ? -k[2] : k[2];
                const double kyz = (fy != fz) ? -k[4] : k[4];
                h0 = make_double2(kxx * m0.x + kxy * m1.x + kxz * m2.x, kxx * m0.y + kxy * m1.y + kxz * m2.y);
                h1 = make_double2(kxy * m0.x + kyy * m1.x + kyz * m2.x, kxy * m0.y + kyy * m1.y + kyz * m2.y);
                h2 = make_double2(kxz * m0.x + kyz * m1.x + kzz * m2.x, kxz * m0.y + kyz * m1.y + kzz * m2.y);
            } else {
                const double2* k = KS + (e * NK + kl) * KCH;
                h0 = cadd(cadd(cmul(k[0], m0), cmul(k[1], m1)), cmul(k[2], m2));
                h1 = cadd(cadd(cmul(k[1], m0), cmul(k[3], m1)), cmul(k[4], m2));
                h2 = cadd(cadd(cmul(k[2], m0), cmul(k[4], m1)), cmul(k[5], m2));
            }
            const double s = a.scale;
            X[i0] = make_double2(h0.x * s, h0.y * s);
            X[i0 + 1] = make_double2(h1.x * s, h1.y * s);
            X[i0 + 2] = make_double2(h2.x * s, h2.y * s);
        }
        __syncthreads();
        if (nxt < ntiles) prefetch_k(nxt);   // KS is free from here on
#pragma unroll
        for (int m = 0; m < R; ++m) v[m] = X[sidx<true, L, R, NL>(b, t + m * TPL)];
        fft_core<L, R, NL, true, 1>(v, X, b, t, tw);
        const int kx = kx0 + b / 3, c = b % 3;
        if (kx < a.hx) {
            double2* line = a.X + g * a.GS + (long long)kx * 3 + c;
#pragma unroll
            for (int i = 0; i < R; ++i) {
                const int e = out_elem<L, R>(t, i);
                if (e < a.n) line[e * a.ES] = v[i];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// x rows: r2c of real length 2M through a complex FFT of length M
// ---------------------------------------------------------------------------
template <int M, bool PM>
__global__ void __launch_bounds__(3 * Cfg<M>::NRr * Cfg<M>::TPL, 2)
k_r2c_fast(const double* __restrict__ in, long long cstride, int pitch, int n_in2,
           double2* __restrict__ out, int CH, int CHP, long long BLKE, long long nrows,
           const double2* __restrict__ twM, const double2* __restrict__ tw2M,
           const int* __restrict__ halt) {
    if (halt && *halt) return;
    constexpr int R = Cfg<M>::R, TPL = Cfg<M>::TPL, NR = Cfg<M>::NRr, NL = 3 * NR;
    constexpr int HX = M + 1;
    extern __shared__ double2 sm[];
    double2* X = sm;
    double2* S = sm + smem_elems<M, R, NL>();
    const long long ntiles = (nrows + NR - 1) / NR;
    const int T = blockDim.x;
    auto prefetch = [&](long long tile) {
        for (int u = threadIdx.x; u < NL * n_in2; u += T) {
            const int bb = u / n_in2, e = u - bb * n_in2;
            const long long row = tile * NR + bb / 3;
            const int c = bb % 3;
            const bool ok = row < nrows;
            cp_async16(&S[u], in + c * cstride + (ok ? row : 0) * pitch + 2 * e, ok);
        }
        cp_async_commit();
    };
    long long tile = blockIdx.x;
    if (tile < ntiles) prefetch(tile);
    const int t = threadIdx.x % TPL, b = threadIdx.x / TPL;
    for (; tile < ntiles; tile += gridDim.x) {
        cp_async_wait_all();
        __syncthreads();
        double2 v[R];
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const int e = t + m * TPL;   // packed pair (x[2e], x[2e+1])
            v[m] = e < n_in2 ? S[b * n_in2 + e] : make_double2(0.0, 0.0);
        }
        __syncthreads();
        const long long nxt = tile + gridDim.x;
        if (nxt < ntiles) prefetch(nxt);
        fft_core<M, R, NL, false, -1>(v, X, b, t, twM);
        if (M > R) __syncthreads();
#pragma unroll
        for (int i = 0; i < R; ++i) X[sidx<false, M, R, NL>(b, out_elem<M, R>(t, i))] = v[i];
        __syncthreads();
        for (int u = threadIdx.x; u < NR * HX * 3; u += T) {
            // row-major output: walk (row, kx, c) so a warp writes along kx; plane-major
            // (CH = 1): walk (kx, row, c) so each plane gets NR*48 contiguous bytes
            int url, kx, cc;
            if (PM) {   // CH == 1
                kx = u / (NR * 3);
                const int r = u - kx * (NR * 3);
                url = r / 3;
                cc = r - 3 * url;
            } else {
                url = u / (HX * 3);
                const int qq = u - url * (HX * 3);
                kx = qq / 3;
                cc = qq - 3 * kx;
            }
            const long long urow = tile * NR + url;
            if (urow >= nrows) continue;
            const int ub = 3 * url + cc;
            const double2 zk = X[sidx<false, M, R, NL>(ub, kx & (M - 1))];
            const double2 zm = X[sidx<false, M, R, NL>(ub, (M - kx) & (M - 1))];
            // E = (Zk + conj Zm)/2, O = (Zk - conj Zm)/(2i), X = E + W^k O
            const double2 E = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
            const double2 O = make_double2(0.5 * (zk.y + zm.y), -0.5 * (zk.x - zm.x));
            const int blk = kx / CH, kxc = kx - blk * CH;
            out[blk * BLKE + (urow * CHP + kxc) * 3 + cc] = cadd(E, cmul(tw2M[kx], O));
        }
    }
}

template <int M, bool PM>
__global__ void __launch_bounds__(3 * Cfg<M>::NRr * Cfg<M>::TPL, 2)
k_c2r_fast(const double2* __restrict__ Xin, int CH, int CHP, long long BLKE, double* __restrict__ out,
           long long cstride, int pitch, int n_out2, long long nrows, const double2* __restrict__ twM,
           const double2* __restrict__ tw2M, const int* __restrict__ halt) {
    if (halt && *halt) return;
    constexpr int R = Cfg<M>::R, TPL = Cfg<M>::TPL, NR = Cfg<M>::NRr, NL = 3 * NR;
    constexpr int HX = M + 1;
    extern __shared__ double2 sm[];
    double2* X = sm;
    double2* S = sm + smem_elems<M, R, NL>();   // NR rows x HX x 3
    const long long ntiles = (nrows + NR - 1) / NR;
    const int T = blockDim.x;
    auto prefetch = [&](long long tile) {
        for (int u = threadIdx.x; u < NR * HX * 3; u += T) {
            // staged as S[url][kx][c]; plane-major input (CH = 1) is read kx-major so
            // consecutive threads fetch contiguous bytes of one plane
            int url, kx, cc;
            if (PM) {   // CH == 1
                kx = u / (NR * 3);
                const int r = u - kx * (NR * 3);
                url = r / 3;
                cc = r - 3 * url;
            } else {
                url = u / (HX * 3);
                const int qq = u - url * (HX * 3);
                kx = qq / 3;
                cc = qq - 3 * kx;
            }
            const long long row = tile * NR + url;
            const bool ok = row < nrows;
            const int blk = kx / CH;
            const long long src = blk * BLKE + ((ok ? row : 0) * CHP + (kx - blk * CH)) * 3 + cc;
            cp_async16(&S[(url * HX + kx) * 3 + cc], Xin + src, ok);
        }
        cp_async_commit();
    };
    long long tile = blockIdx.x;
    if (tile < ntiles) prefetch(tile);
    const int t = threadIdx.x % TPL, b = threadIdx.x / TPL;
    const int rl = b / 3, c = b - 3 * rl;
    for (; tile < ntiles; tile += gridDim.x) {
        cp_async_wait_all();
        __syncthreads();
        double2 v[R];
        const double2* srow = S + rl * HX * 3 + c;
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const int k = t + m * TPL;
            const double2 xk = srow[3 * k];
            const double2 xm = srow[3 * (M - k)];
            // Z = (Xk + conj Xm) + i (Xk - conj Xm) W^-k
            const double2 A = make_double2(xk.x + xm.x, xk.y - xm.y);
            const double2 Bm = make_double2(xk.x - xm.x, xk.y + xm.y);
            const double2 w = tw2M[k];
            const double2 B = cmul(Bm, make_double2(w.x, -w.y));
            v[m] = make_double2(A.x - B.y, A.y + B.x);
        }
        __syncthreads();
        const long long nxt = tile + gridDim.x;
        if (nxt < ntiles) prefetch(nxt);
        fft_core<M, R, NL, false, 1>(v, X, b, t, twM);
        const long long row = tile * NR + rl;
        if (row < nrows) {
            double2* dst = reinterpret_cast<double2*>(out + c * cstride + row * pitch);
#pragma unroll
            for (int i = 0; i < R; ++i) {
                const int e = out_elem<M, R>(t, i);
                if (e < n_out2) dst[e] = v[i];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// launch helpers: persistent grids sized by occupancy
// ---------------------------------------------------------------------------
static bool pow2(int v) { return v >= 2 && (v & (v - 1)) == 0; }

static const size_t kFastSmemMax = 220 * 1024;

static int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// grid size for a persistent kernel (cached per kernel and shared-memory size)
template <class F>
static int persistent_grid(F f, int threads, size_t smem, long long ntiles, int* grid) {
    static std::mutex mu;
    static std::set<const void*> attr_done;
    static std::map<std::pair<const void*, size_t>, int> occ;
    std::lock_guard<std::mutex> lk(mu);
    if (!attr_done.count((const void*)f)) {
        MXB_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFastSmemMax));
        MXB_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        attr_done.insert((const void*)f);
    }
    auto key = std::make_pair((const void*)f, smem);
    auto it = occ.find(key);
    int per_sm;
    if (it == occ.end()) {
        MXB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, threads, smem));
        occ[key] = per_sm;
    } else {
        per_sm = it->second;
    }
    if (per_sm < 1) { set_error("fast FFT kernel does not fit on an SM"); return MXB_EINVAL; }
    const long long cap = (long long)per_sm * num_sms();
    *grid = (int)(ntiles < cap ? ntiles : cap);
    return MXB_OK;
}

template <int L, int RM, int NLD>
static int col_staged(int dir, const ColArgs& a, const double2* tw, cudaStream_t st, const int* halt) {
    constexpr int R = Cfg<L, RM>::R, NL = Cfg<L, RM>::NLc / NLD;
    const size_t sm = ((size_t)smem_elems<L, R, NL>() + (size_t)NL * a.n_in) * sizeof(double2);
    const long long ntiles = (a.nlines + NL - 1) / NL;
    const int thr = NL * Cfg<L, RM>::TPL;
    int grid = 0, rc;
    if (dir < 0) {
        if ((rc = persistent_grid(k_col_fast<L, -1, RM, NLD>, thr, sm, ntiles, &grid))) return rc;
        k_col_fast<L, -1, RM, NLD><<<grid, thr, sm, st>>>(a, tw, halt);
    } else {
        if ((rc = persistent_grid(k_col_fast<L, 1, RM, NLD>, thr, sm, ntiles, &grid))) return rc;
        k_col_fast<L, 1, RM, NLD><<<grid, thr, sm, st>>>(a, tw, halt);
    }
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

template <int L, int RM>
static int col_launch(int dir, const ColArgs& a, const double2* tw, cudaStream_t st, const int* halt) {
    constexpr int R = Cfg<L, RM>::R, NL = Cfg<L, RM>::NLc;
    const size_t full = ((size_t)smem_elems<L, R, NL>() + (size_t)NL * a.n_in) * sizeof(double2);
    // staged (cp.async prefetch of the next tile) whenever two CTAs fit on an SM;
    // halve the lines per CTA for long inputs (the inverse pass reads all L rows)
    if (full <= 110 * 1024) return col_staged<L, RM, 1>(dir, a, tw, st, halt);
    if (NL >= 4) {
        const size_t half = ((size_t)smem_elems<L, R, NL / 2>() + (size_t)(NL / 2) * a.n_in) * sizeof(double2);
        if (half <= 110 * 1024) return col_staged<L, RM, 2>(dir, a, tw, st, halt);
    }
    const long long ntiles = (a.nlines + NL - 1) / NL;
    const int thr = NL * Cfg<L, RM>::TPL;
    int grid = 0, rc;
    const size_t smd = (size_t)smem_elems<L, R, NL>() * sizeof(double2);
    if (smd > kFastSmemMax) return -1;
    if (dir < 0) {
        if ((rc = persistent_grid(k_col_direct<L, -1, RM>, thr, smd, 1, &grid))) return rc;
        k_col_direct<L, -1, RM><<<(unsigned)ntiles, thr, smd, st>>>(a, tw, halt);
    } else {
        if ((rc = persistent_grid(k_col_direct<L, 1, RM>, thr, smd, 1, &grid))) return rc;
        k_col_direct<L, 1, RM><<<(unsigned)ntiles, thr, smd, st>>>(a, tw, halt);
    }
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

template <int L, int RM>
static int fused_launch(int kmode, const FusedArgs& a, const double2* tw, cudaStream_t st,
                        const int* halt) {
    constexpr int R = Cfg<L, RM>::R, NK = Cfg<L, RM>::NKf, NL = 3 * NK;
    const int krows = (kmode == 2 || kmode == 4) ? (L / 2 + 1) : L;
    const int kch = (kmode == 2 || kmode == 4) ? 3 : 6;
    const size_t sm = ((size_t)smem_elems<L, R, NL>() + (size_t)NL * a.n + (size_t)krows * NK * kch) *
                      sizeof(double2);
    if (sm > kFastSmemMax) return -1;
    const long long ntiles = (long long)a.G * ((a.hx + NK - 1) / NK);
    const int thr = NL * Cfg<L, RM>::TPL;
    int grid = 0, rc;
    if (kmode == 2) {
        if ((rc = persistent_grid(k_fused_fast<L, 2, RM>, thr, sm, ntiles, &grid))) return rc;
        k_fused_fast<L, 2, RM><<<grid, thr, sm, st>>>(a, tw, halt);
    } else if (kmode == 4) {
        if ((rc = persistent_grid(k_fused_fast<L, 4, RM>, thr, sm, ntiles, &grid))) return rc;
        k_fused_fast<L, 4, RM><<<grid, thr, sm, st>>>(a, tw, halt);
    } else {
        if ((rc = persistent_grid(k_fused_fast<L, 0, RM>, thr, sm, ntiles, &grid))) return rc;
        k_fused_fast<L, 0, RM><<<grid, thr, sm, st>>>(a, tw, halt);
    }
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

template <int M>
static int rows_launch(bool fwd, const double* in_r, double2* X, double* out_r, long long cstride,
                       int pitch, int nhalf, int CH, int CHP, long long BLKE, long long nrows,
                       const double2* twM, const double2* tw2M, cudaStream_t st, const int* halt) {
    constexpr int R = Cfg<M>::R, NR = Cfg<M>::NRr, NL = 3 * NR;
    const size_t stage = fwd ? (size_t)NL * nhalf : (size_t)NR * (M + 1) * 3;
    const size_t sm = ((size_t)smem_elems<M, R, NL>() + stage) * sizeof(double2);
    if (sm > kFastSmemMax) return -1;
    const long long ntiles = (nrows + NR - 1) / NR;
    const int thr = NL * Cfg<M>::TPL;
    int grid = 0, rc;
    // plane-major layout (one kx per block, CH = 1): walk kx-major
    if (fwd && CH == 1) {
        if ((rc = persistent_grid(k_r2c_fast<M, true>, thr, sm, ntiles, &grid))) return rc;
        k_r2c_fast<M, true><<<grid, thr, sm, st>>>(in_r, cstride, pitch, nhalf, X, CH, CHP, BLKE, nrows, twM,
                                                   tw2M, halt);
    } else if (fwd) {
        if ((rc = persistent_grid(k_r2c_fast<M, false>, thr, sm, ntiles, &grid))) return rc;
        k_r2c_fast<M, false><<<grid, thr, sm, st>>>(in_r, cstride, pitch, nhalf, X, CH, CHP, BLKE, nrows, twM,
                                                    tw2M, halt);
    } else if (CH == 1) {
        if ((rc = persistent_grid(k_c2r_fast<M, true>, thr, sm, ntiles, &grid))) return rc;
        k_c2r_fast<M, true><<<grid, thr, sm, st>>>(X, CH, CHP, BLKE, out_r, cstride, pitch, nhalf, nrows, twM,
                                                   tw2M, halt);
    } else {
        if ((rc = persistent_grid(k_c2r_fast<M, false>, thr, sm, ntiles, &grid))) return rc;
        k_c2r_fast<M, false><<<grid, thr, sm, st>>>(X, CH, CHP, BLKE, out_r, cstride, pitch, nhalf, nrows, twM,
                                                    tw2M, halt);
    }
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

#define MXB_POW2_CASES(MACRO) \
    MACRO(2) MACRO(4) MACRO(8) MACRO(16) MACRO(32) MACRO(64) MACRO(128) MACRO(256) MACRO(512) \
    MACRO(1024) MACRO(2048) MACRO(4096)

// each returns -1 when the fast path does not cover the shape
// radix of the register-resident kernels (MXB_COL_RADIX / MXB_FUSED_RADIX = 8 or 16)
static int env_radix(const char* name, int dflt) {
    const char* v = getenv(name);
    if (!v) return dflt;
    const int r = atoi(v);
    return (r == 8 || r == 16) ? r : dflt;
}
static int col_radix() { static int r = env_radix("MXB_COL_RADIX", 16); return r; }
static int fused_radix() { static int r = env_radix("MXB_FUSED_RADIX", 16); return r; }

int fast_cols(int dir, int L, const double2* in, double2* out, int n_in, int n_out,
              long long ES_in, long long ES_out, int Q, long long nlines, long long OS_in,
              long long OS_out, const double2* tw, cudaStream_t st, const int* halt) {
    if (!pow2(L)) return -1;
    const ColArgs a{in, out, n_in, n_out, ES_in, ES_out, Q, nlines, OS_in, OS_out};
    if (col_radix() == 8) {
#define CASE(V) case V: return col_launch<V, 8>(dir, a, tw, st, halt);
        switch (L) { MXB_POW2_CASES(CASE) default: return -1; }
#undef CASE
    }
#define CASE(V) case V: return col_launch<V, 16>(dir, a, tw, st, halt);
    switch (L) { MXB_POW2_CASES(CASE) default: return -1; }
#undef CASE
}

bool fast_fused_ok(int L) { return L == 1 || (pow2(L) && L <= 1024); }

int fast_fused(int L, int kmode, const FusedArgs& a, const double2* tw, cudaStream_t st,
               const int* halt) {
    if (!fast_fused_ok(L) || kmode == 1) return -1;
    if (fused_radix() == 8) {
#define CASE(V) case V: return fused_launch<V, 8>(kmode, a, tw, st, halt);
        switch (L) {
            CASE(1) CASE(2) CASE(4) CASE(8) CASE(16) CASE(32) CASE(64) CASE(128) CASE(256) CASE(512)
            CASE(1024) CASE(2048)
            default: return -1;
        }
#undef CASE
    }
#define CASE(V) case V: return fused_launch<V, 16>(kmode, a, tw, st, halt);
    switch (L) {
        CASE(1) CASE(2) CASE(4) CASE(8) CASE(16) CASE(32) CASE(64) CASE(128) CASE(256) CASE(512)
        CASE(1024) CASE(2048)
        default: return -1;
    }
#undef CASE
}

int fast_rows(bool fwd, int M, const double* in_r, double2* X, double* out_r, long long cstride,
              int pitch, int nhalf, int CH, int CHP, long long BLKE, long long nrows,
              const double2* twM, const double2* tw2M, cudaStream_t st, const int* halt) {
    if (!pow2(M)) return -1;
    const int rw = warp_rows(fwd, M, in_r, X, out_r, cstride, pitch, nhalf, CH, CHP, BLKE, nrows, twM, tw2M, st, halt);
    if (rw != -1) return rw;
#define CASE(V) case V: return rows_launch<V>(fwd, in_r, X, out_r, cstride, pitch, nhalf, CH, CHP, BLKE, nrows, twM, tw2M, st, halt);
    switch (M) { MXB_POW2_CASES(CASE) default: return -1; }
#undef CASE
}

}  // namespace mxb
