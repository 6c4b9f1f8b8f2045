// Fast-path kernels of the demag pipeline for power-of-two padded lengths
// (register-resident radix-16 Stockham, fft_fast.cuh).  Same pass structure
// and buffer layouts as the generic kernels in demag.cu:
//   x rows  : real r2c / c2r of length px via one complex FFT of length px/2
//   columns : strided c2c lines (y passes), lines fastest in shared memory
//   fused   : forward c2c * 3x3 kernel multiply * inverse c2c (z, or y for films)
#include <mutex>
#include <set>
#include <utility>

#include "demag.cuh"
#include "fft_fast.cuh"

namespace mxb {

using namespace ff;

template <int L> struct Cfg {
    static constexpr int R = L >= 16 ? 16 : (L < 1 ? 1 : L);
    static constexpr int TPL = L / R;
    // columns: ~256 threads, at least 2 lines (32-byte segments)
    static constexpr int NLc = (256 * R / L) >= 2 ? (256 * R / L) : 2;
    // fused: NK kx columns x 3 components (one kx column for long lines, so
    // two or three CTAs share an SM and overlap their load/compute phases)
    static constexpr int NKf = L >= 512 ? 1 : ((256 * R / (3 * L)) >= 2 ? (256 * R / (3 * L)) : 2);
    // rows (M = L complex points per row): NR rows x 3 components
    static constexpr int NRr = (256 * R / (3 * L)) >= 1 ? (256 * R / (3 * L)) : 1;
};

// ---------------------------------------------------------------------------
// strided columns (y passes)
// ---------------------------------------------------------------------------
template <int L, int DIR>
__global__ void __launch_bounds__(Cfg<L>::NLc * Cfg<L>::TPL, 2)
k_col_fast(const double2* in, double2* out, int n_in, int n_out, long long ES_in, long long ES_out,
           int Q, long long nlines, long long OS_in, long long OS_out,
           const double2* __restrict__ tw, const int* __restrict__ halt) {
    if (halt && *halt) return;
    constexpr int R = Cfg<L>::R, TPL = Cfg<L>::TPL, NL = Cfg<L>::NLc;
    extern __shared__ double2 sm[];
    const int b = threadIdx.x % NL, t = threadIdx.x / NL;
    const long long g = (long long)blockIdx.x * NL + b;
    const bool ok = g < nlines;
    const long long o = ok ? g / Q : 0, q = ok ? g - o * Q : 0;
    const double2* src = in + o * OS_in + q;
    double2 v[R];
#pragma unroll
    for (int m = 0; m < R; ++m) {
        const int e = t + m * TPL;
        v[m] = (ok && e < n_in) ? src[e * ES_in] : make_double2(0.0, 0.0);
    }
    fft_core<L, R, NL, true, DIR>(v, sm, b, t, tw);
    double2* dst = out + o * OS_out + q;
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const int e = out_elem<L, R>(t, i);
        if (ok && e < n_out) dst[e * ES_out] = v[i];
    }
}

// ---------------------------------------------------------------------------
// fused forward * multiply * inverse along the outer axis
// K layouts: KMODE 0 complex [e*G+g][kx][6]; 1 real same; 2 real quarter
// [e'][g'][kx][6] with e' = min(e, L-e), g' = min(g, G-g) and parity signs.
// ---------------------------------------------------------------------------

template <int KMODE>
__device__ __forceinline__ void kernel6(const FusedArgs& a, int L, int e, int g, int kx, double2 k[6]) {
    if (KMODE == 0) {
        const double2* p = (const double2*)a.K + (((long long)e * a.G + g) * a.hxp + kx) * 6;
#pragma unroll
        for (int c = 0; c < 6; ++c) k[c] = p[c];
    } else if (KMODE == 1) {
        const double* p = (const double*)a.K + (((long long)e * a.G + g) * a.hxp + kx) * 6;
#pragma unroll
        for (int c = 0; c < 6; ++c) k[c] = make_double2(p[c], 0.0);
    } else {
        const bool re = 2 * e > L, rg = 2 * g > a.G;
        const int e2 = re ? L - e : e, g2 = rg ? a.G - g : g;
        const int G2 = a.G / 2 + 1;
        const double* p = (const double*)a.K + (((long long)e2 * G2 + g2) * a.hxp + kx) * 6;
        // reflected axes: e is z (3-D) or y (film); g is y (3-D) or z (film, size 1)
        const bool fy = a.e_is_z ? rg : re;
        const bool fz = a.e_is_z ? re : rg;
        const double sxy = fy ? -1.0 : 1.0;
        const double sxz = fz ? -1.0 : 1.0;
        const double syz = (fy != fz) ? -1.0 : 1.0;
        k[0] = make_double2(p[0], 0.0);
        k[1] = make_double2(sxy * p[1], 0.0);
        k[2] = make_double2(sxz * p[2], 0.0);
        k[3] = make_double2(p[3], 0.0);
        k[4] = make_double2(syz * p[4], 0.0);
        k[5] = make_double2(p[5], 0.0);
    }
}

template <int L, int KMODE>
__global__ void __launch_bounds__(3 * Cfg<L>::NKf * Cfg<L>::TPL, 2)
k_fused_fast(FusedArgs a, const double2* __restrict__ tw, const int* __restrict__ halt) {
    if (halt && *halt) return;
    constexpr int R = Cfg<L>::R, TPL = Cfg<L>::TPL, NK = Cfg<L>::NKf, NL = 3 * NK;
    extern __shared__ double2 sm[];
    const int b = threadIdx.x % NL, t = threadIdx.x / NL;
    const int g = blockIdx.y;
    const int kl = b / 3, c = b - 3 * kl;
    const int kx = blockIdx.x * NK + kl;
    const bool ok = kx < a.hx;
    double2* line = a.X + g * a.GS + (long long)kx * 3 + c;
    double2 v[R];
#pragma unroll
    for (int m = 0; m < R; ++m) {
        const int e = t + m * TPL;
        v[m] = (ok && e < a.n) ? line[e * a.ES] : make_double2(0.0, 0.0);
    }
    fft_core<L, R, NL, true, -1>(v, sm, b, t, tw);
    // spectra to shared memory in natural order, then the 3x3 multiply per point
    if (L > R) __syncthreads();
#pragma unroll
    for (int i = 0; i < R; ++i) sm[sidx<true, L, R, NL>(b, out_elem<L, R>(t, i))] = v[i];
    __syncthreads();
    for (int u = threadIdx.x; u < NK * L; u += blockDim.x) {
        const int ul = u % NK, e = u / NK;
        const int ukx = blockIdx.x * NK + ul;
        if (ukx >= a.hx) continue;
        double2 k[6];
        kernel6<KMODE>(a, L, e, g, ukx, k);
        const int i0 = sidx<true, L, R, NL>(3 * ul, e);
        const double2 m0 = sm[i0], m1 = sm[i0 + 1], m2 = sm[i0 + 2];
        double2 h0, h1, h2;
        if (KMODE == 0) {
            h0 = cadd(cadd(cmul(k[0], m0), cmul(k[1], m1)), cmul(k[2], m2));
            h1 = cadd(cadd(cmul(k[1], m0), cmul(k[3], m1)), cmul(k[4], m2));
            h2 = cadd(cadd(cmul(k[2], m0), cmul(k[4], m1)), cmul(k[5], m2));
        } else {
            const double kxx = k[0].x, kxy = k[1].x, kxz = k[2].x, kyy = k[3].x, kyz = k[4].x, kzz = k[5].x;
            h0 = make_double2(kxx * m0.x + kxy * m1.x + kxz * m2.x, kxx * m0.y + kxy * m1.y + kxz * m2.y);
            h1 = make_double2(kxy * m0.x + kyy * m1.x + kyz * m2.x, kxy * m0.y + kyy * m1.y + kyz * m2.y);
            h2 = make_double2(kxz * m0.x + kyz * m1.x + kzz * m2.x, kxz * m0.y + kyz * m1.y + kzz * m2.y);
        }
        const double s = a.scale;
        sm[i0] = make_double2(h0.x * s, h0.y * s);
        sm[i0 + 1] = make_double2(h1.x * s, h1.y * s);
        sm[i0 + 2] = make_double2(h2.x * s, h2.y * s);
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < R; ++m) v[m] = sm[sidx<true, L, R, NL>(b, t + m * TPL)];
    fft_core<L, R, NL, true, 1>(v, sm, b, t, tw);
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const int e = out_elem<L, R>(t, i);
        if (ok && e < a.n) line[e * a.ES] = v[i];
    }
}

// ---------------------------------------------------------------------------
// x rows: r2c of real length 2M through a complex FFT of length M
// ---------------------------------------------------------------------------
template <int M>
__global__ void __launch_bounds__(3 * Cfg<M>::NRr * Cfg<M>::TPL, 2)
k_r2c_fast(const double* __restrict__ in, long long cstride, int pitch, int n_in2,
           double2* __restrict__ out, int hxp, long long nrows, const double2* __restrict__ twM,
           const double2* __restrict__ tw2M, const int* __restrict__ halt) {
    if (halt && *halt) return;
    constexpr int R = Cfg<M>::R, TPL = Cfg<M>::TPL, NR = Cfg<M>::NRr, NL = 3 * NR;
    extern __shared__ double2 sm[];
    const int t = threadIdx.x % TPL, b = threadIdx.x / TPL;
    const int rl = b / 3, c = b - 3 * rl;
    const long long row = (long long)blockIdx.x * NR + rl;
    const bool ok = row < nrows;
    const double2* src = reinterpret_cast<const double2*>(in + c * cstride + row * pitch);
    double2 v[R];
#pragma unroll
    for (int m = 0; m < R; ++m) {
        const int e = t + m * TPL;   // packed pair (x[2e], x[2e+1])
        v[m] = (ok && e < n_in2) ? src[e] : make_double2(0.0, 0.0);
    }
    fft_core<M, R, NL, false, -1>(v, sm, b, t, twM);
    if (M > R) __syncthreads();
#pragma unroll
    for (int i = 0; i < R; ++i) sm[sidx<false, M, R, NL>(b, out_elem<M, R>(t, i))] = v[i];
    __syncthreads();
    constexpr int HX = M + 1;
    for (int u = threadIdx.x; u < NR * HX * 3; u += blockDim.x) {
        const int url = u / (HX * 3), qq = u - url * (HX * 3);
        const int kx = qq / 3, cc = qq - 3 * kx;
        const long long urow = (long long)blockIdx.x * NR + url;
        if (urow >= nrows) continue;
        const int ub = 3 * url + cc;
        const double2 zk = sm[sidx<false, M, R, NL>(ub, kx & (M - 1))];
        const double2 zm = sm[sidx<false, M, R, NL>(ub, (M - kx) & (M - 1))];
        // E = (Zk + conj Zm)/2, O = (Zk - conj Zm)/(2i), X = E + W^k O
        const double2 E = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
        const double2 O = make_double2(0.5 * (zk.y + zm.y), -0.5 * (zk.x - zm.x));
        const double2 w = tw2M[kx];
        const double2 X = cadd(E, cmul(w, O));
        out[(urow * hxp + kx) * 3 + cc] = X;
    }
}

template <int M>
__global__ void __launch_bounds__(3 * Cfg<M>::NRr * Cfg<M>::TPL, 2)
k_c2r_fast(const double2* __restrict__ X, int hxp, double* __restrict__ out, long long cstride,
           int pitch, int n_out2, long long nrows, const double2* __restrict__ twM,
           const double2* __restrict__ tw2M, const int* __restrict__ halt) {
    if (halt && *halt) return;
    constexpr int R = Cfg<M>::R, TPL = Cfg<M>::TPL, NR = Cfg<M>::NRr, NL = 3 * NR;
    constexpr int HX = M + 1;
    extern __shared__ double2 sm[];
    double2* nyq = sm + smem_elems<M, R, NL>();
    for (int u = threadIdx.x; u < NR * HX * 3; u += blockDim.x) {
        const int url = u / (HX * 3), qq = u - url * (HX * 3);
        const int kx = qq / 3, cc = qq - 3 * kx;
        const long long urow = (long long)blockIdx.x * NR + url;
        const double2 x = urow < nrows ? X[(urow * hxp + kx) * 3 + cc] : make_double2(0.0, 0.0);
        if (kx < M) sm[sidx<false, M, R, NL>(3 * url + cc, kx)] = x;
        else nyq[3 * url + cc] = x;
    }
    __syncthreads();
    const int t = threadIdx.x % TPL, b = threadIdx.x / TPL;
    const int rl = b / 3, c = b - 3 * rl;
    const long long row = (long long)blockIdx.x * NR + rl;
    double2 v[R];
#pragma unroll
    for (int m = 0; m < R; ++m) {
        const int k = t + m * TPL;
        const double2 xk = sm[sidx<false, M, R, NL>(b, k)];
        const double2 xm = k == 0 ? nyq[b] : sm[sidx<false, M, R, NL>(b, M - k)];
        // Z = (Xk + conj Xm) + i (Xk - conj Xm) W^-k
        const double2 A = make_double2(xk.x + xm.x, xk.y - xm.y);
        const double2 Bm = make_double2(xk.x - xm.x, xk.y + xm.y);
        const double2 w = tw2M[k];
        const double2 B = cmul(Bm, make_double2(w.x, -w.y));
        v[m] = make_double2(A.x - B.y, A.y + B.x);
    }
    fft_core<M, R, NL, false, 1>(v, sm, b, t, twM);
    if (row < nrows) {
        double2* dst = reinterpret_cast<double2*>(out + c * cstride + row * pitch);
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int e = out_elem<M, R>(t, i);
            if (e < n_out2) dst[e] = v[i];
        }
    }
}

// ---------------------------------------------------------------------------
// dispatch
// ---------------------------------------------------------------------------
static bool pow2(int v) { return v >= 2 && (v & (v - 1)) == 0; }

static const size_t kFastSmemMax = 200 * 1024;

template <class F>
static int set_attr(F f, size_t bytes) {
    // one attribute call per kernel (per device)
    static std::mutex mu;
    static std::set<std::pair<int, const void*>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    if (done.count({dev, (const void*)f})) return MXB_OK;
    (void)bytes;
    MXB_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFastSmemMax));
    done.insert({dev, (const void*)f});
    return MXB_OK;
}

template <int L>
static int col_launch(int dir, const double2* in, double2* out, int n_in, int n_out, long long ES_in,
                      long long ES_out, int Q, long long nlines, long long OS_in, long long OS_out,
                      const double2* tw, cudaStream_t st, const int* halt) {
    constexpr int R = Cfg<L>::R, NL = Cfg<L>::NLc;
    const size_t sm = (size_t)smem_elems<L, R, NL>() * sizeof(double2);
    if (sm > kFastSmemMax) return -1;
    const unsigned nb = (unsigned)((nlines + NL - 1) / NL);
    const int thr = NL * Cfg<L>::TPL;
    if (dir < 0) {
        int rc = set_attr(k_col_fast<L, -1>, sm);
        if (rc) return rc;
        k_col_fast<L, -1><<<nb, thr, sm, st>>>(in, out, n_in, n_out, ES_in, ES_out, Q, nlines, OS_in,
                                              OS_out, tw, halt);
    } else {
        int rc = set_attr(k_col_fast<L, 1>, sm);
        if (rc) return rc;
        k_col_fast<L, 1><<<nb, thr, sm, st>>>(in, out, n_in, n_out, ES_in, ES_out, Q, nlines, OS_in,
                                             OS_out, tw, halt);
    }
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

template <int L>
static int fused_launch(int kmode, const FusedArgs& a, const double2* tw, cudaStream_t st,
                        const int* halt) {
    constexpr int R = Cfg<L>::R, NK = Cfg<L>::NKf, NL = 3 * NK;
    const size_t sm = (size_t)smem_elems<L, R, NL>() * sizeof(double2);
    if (sm > kFastSmemMax) return -1;
    dim3 grid((a.hx + NK - 1) / NK, a.G);
    const int thr = NL * Cfg<L>::TPL;
    int rc;
    switch (kmode) {
        case 0:
            if ((rc = set_attr(k_fused_fast<L, 0>, sm))) return rc;
            k_fused_fast<L, 0><<<grid, thr, sm, st>>>(a, tw, halt);
            break;
        case 1:
            if ((rc = set_attr(k_fused_fast<L, 1>, sm))) return rc;
            k_fused_fast<L, 1><<<grid, thr, sm, st>>>(a, tw, halt);
            break;
        default:
            if ((rc = set_attr(k_fused_fast<L, 2>, sm))) return rc;
            k_fused_fast<L, 2><<<grid, thr, sm, st>>>(a, tw, halt);
    }
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

template <int M>
static int rows_launch(bool fwd, const double* in_r, double2* X, double* out_r, long long cstride,
                       int pitch, int nhalf, int hxp, long long nrows, const double2* twM,
                       const double2* tw2M, cudaStream_t st, const int* halt) {
    constexpr int R = Cfg<M>::R, NR = Cfg<M>::NRr, NL = 3 * NR;
    const size_t sm = ((size_t)smem_elems<M, R, NL>() + NL) * sizeof(double2);
    if (sm > kFastSmemMax) return -1;
    const unsigned nb = (unsigned)((nrows + NR - 1) / NR);
    const int thr = NL * Cfg<M>::TPL;
    int rc;
    if (fwd) {
        if ((rc = set_attr(k_r2c_fast<M>, sm))) return rc;
        k_r2c_fast<M><<<nb, thr, sm, st>>>(in_r, cstride, pitch, nhalf, X, hxp, nrows, twM, tw2M, halt);
    } else {
        if ((rc = set_attr(k_c2r_fast<M>, sm))) return rc;
        k_c2r_fast<M><<<nb, thr, sm, st>>>(X, hxp, out_r, cstride, pitch, nhalf, nrows, twM, tw2M, halt);
    }
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

#define MXB_POW2_CASES(MACRO) \
    MACRO(2) MACRO(4) MACRO(8) MACRO(16) MACRO(32) MACRO(64) MACRO(128) MACRO(256) MACRO(512) \
    MACRO(1024) MACRO(2048) MACRO(4096)

// returns -1 when the fast path does not cover this shape
int fast_cols(int dir, int L, const double2* in, double2* out, int n_in, int n_out,
              long long ES_in, long long ES_out, int Q, long long nlines, long long OS_in,
              long long OS_out, const double2* tw, cudaStream_t st, const int* halt) {
    if (!pow2(L)) return -1;
#define CASE(V) case V: return col_launch<V>(dir, in, out, n_in, n_out, ES_in, ES_out, Q, nlines, OS_in, OS_out, tw, st, halt);
    switch (L) { MXB_POW2_CASES(CASE) default: return -1; }
#undef CASE
}

bool fast_fused_ok(int L) { return L == 1 || (pow2(L) && L <= 2048); }

int fast_fused(int L, int kmode, const FusedArgs& a, const double2* tw, cudaStream_t st,
               const int* halt) {
    if (!fast_fused_ok(L)) return -1;
#define CASE(V) case V: return fused_launch<V>(kmode, a, tw, st, halt);
    switch (L) {
        CASE(1) CASE(2) CASE(4) CASE(8) CASE(16) CASE(32) CASE(64) CASE(128) CASE(256) CASE(512)
        CASE(1024) CASE(2048)
        default: return -1;
    }
#undef CASE
}

int fast_rows(bool fwd, int M, const double* in_r, double2* X, double* out_r, long long cstride,
              int pitch, int nhalf, int hxp, long long nrows, const double2* twM,
              const double2* tw2M, cudaStream_t st, const int* halt) {
    if (!pow2(M)) return -1;
#define CASE(V) case V: return rows_launch<V>(fwd, in_r, X, out_r, cstride, pitch, nhalf, hxp, nrows, twM, tw2M, st, halt);
    switch (M) { MXB_POW2_CASES(CASE) default: return -1; }
#undef CASE
}

}  // namespace mxb
