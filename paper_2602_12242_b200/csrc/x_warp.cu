// x passes (P1 r2c / P5 c2r) with the warp-per-line FFT core, for rows of
// nx = 512 reals (px = 1024, one complex FFT of M = 512 per row via the
// half-length packing, as k_r2c_fast / k_c2r_fast in demag_fast.cu).
//
// A CTA is 3 warps, one per component; each warp transforms two rows of its
// component (fw::fft512x2: register DFT-16s, one swizzled transpose,
// register DFT-32s), so a CTA handles a row pair.  The r2c loads its packed
// rows straight into registers (contiguous 16-byte pairs, whole sectors per
// warp) and untangles the half-length spectrum through the warp's tile; the
// outputs go out in 128-bin chunks staged in shared memory so every store
// run is contiguous in either layout.  The c2r stages the spectrum rows of
// its pair with cp.async, forms the packed input, and writes the real rows
// straight from registers.  Layouts: row-major X[row][CHP][3] of one rank
// (CH >= hx) or plane-major X[kx][row][3] (CH = 1, the plane pipeline).
#include <stdlib.h>

#include "demag.cuh"
#include "fft_warp.cuh"
#include "tma.cuh"

namespace mxb {

using namespace ff;

#ifndef MXB_XW_TMA_IN
#define MXB_XW_TMA_IN 1   // r2c input rows staged by TMA bulk copies
#endif

#ifndef MXB_XW_EXIT_READ
#define MXB_XW_EXIT_READ 1
#endif

#ifndef MXB_XW_TWREC   // r2c: untangling twiddles by products of W^32 between table anchors
#define MXB_XW_TWREC 1   // (with the bin-outer untangle loop: r2c 8.81 -> 8.13 ms per step)
#endif

#ifndef MXB_XW_TWPRE   // c2r: untangling twiddles loaded before the TMA wait (6.89 -> 6.81 ms per step)
#define MXB_XW_TWPRE 1
#endif

#ifndef MXB_XW_PFD_DEFAULT   // r2c: L2 prefetch of the input pfd CTAs ahead (148: 8.23 -> 7.71 ms per step)
#define MXB_XW_PFD_DEFAULT 148
#endif

namespace {
constexpr int XM = 512;          // complex FFT length (px / 2)
constexpr int XHX = XM + 1;      // spectrum bins kept (px / 2 + 1)
}

template <bool PM>
__global__ void __launch_bounds__(96, 4)
k_r2c_w(const double* __restrict__ in, long long cstride, int pitch, double2* __restrict__ out, int CHP,
        long long BLKE, const double2* __restrict__ tw512, const double2* __restrict__ tw1024,
        const int* __restrict__ halt, const __grid_constant__ CUtensorMap map_main,
        const __grid_constant__ CUtensorMap map_tail, int pfd) {
    if (halt && *halt) return;
    // 3 x 1024 transpose tiles, then the output pair: [kx][line][c] (plane-major,
    // TMA boxes of 256 planes x 96 B) or [line][kx][c] (row-major, two bulk rows)
    extern __shared__ __align__(128) double2 W[];
    const int c = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double2* Wc = W + c * 1024;
    const long long row0 = 2LL * blockIdx.x;
    double2 a[16], b[16], v[32];
#if MXB_XW_TMA_IN
    // the row pair of each component is 8 KB contiguous (pitch == nx): three
    // bulk copies into the (still free) tile memory, one mbarrier wait
    __shared__ alignas(8) unsigned long long mbar;
    if (threadIdx.x == 0) {
        mbar_init(&mbar);
        mbar_expect(&mbar, 3 * 2 * XM * 8);
        for (int q = 0; q < 3; ++q)
            bulk_g2s_tx(W + q * XM, in + q * cstride + row0 * pitch, 2 * XM * 8, &mbar);
        // the input of the CTA pfd row pairs ahead (about one wave later on this
        // SM slot) into L2, so its staging wait is an L2 hit
        if (pfd && blockIdx.x + pfd < gridDim.x)
            for (int q = 0; q < 3; ++q)
                prefetch_l2(in + q * cstride + (row0 + 2LL * pfd) * pitch, 2 * XM * 8);
    }
    __syncthreads();
    mbar_wait(&mbar, 0);
    {
        const double2* s0 = W + c * XM;
#pragma unroll
        for (int m = 0; m < 16; ++m) {   // packed pairs (x[2n], x[2n+1]), n < 256 non-zero
            a[m] = m < 8 ? s0[lane + 32 * m] : make_double2(0.0, 0.0);
            b[m] = m < 8 ? s0[XM / 2 + lane + 32 * m] : make_double2(0.0, 0.0);
        }
    }
    __syncthreads();   // the staged rows are in registers: the tiles may overwrite them
#else
    const double2* s0 = reinterpret_cast<const double2*>(in + c * cstride + row0 * pitch);
    const double2* s1 = reinterpret_cast<const double2*>(in + c * cstride + (row0 + 1) * pitch);
#pragma unroll
    for (int m = 0; m < 16; ++m) {   // packed pairs (x[2n], x[2n+1]), n < 256 non-zero
        a[m] = m < 8 ? __ldg(s0 + lane + 32 * m) : make_double2(0.0, 0.0);
        b[m] = m < 8 ? __ldg(s1 + lane + 32 * m) : make_double2(0.0, 0.0);
    }
#endif
    fw::fft512x2<-1>(a, b, v, Wc, lane, tw512);   // HALF_IN measured 1% slower here
    // Z_line[k1 + 16 k2] -> tile, natural order per line
    {
        const int line = lane >> 4, k1 = lane & 15;
        __syncwarp();
#pragma unroll
        for (int k2 = 0; k2 < 32; ++k2) Wc[line * XM + k1 + 16 * k2] = v[fw::p32(k2)];
        __syncwarp();
    }
    // untangle all XHX bins of both lines into registers (bin kx = lane + 32 i)
    constexpr int NI = (XHX + 31) / 32;   // 17
    double2 xo[2][NI];
#if MXB_XW_TWREC
    // W^kx for kx = lane + 32 i: table anchors every 4th i, products with the exact
    // W^32 in between (5 + 1 loads per lane instead of 17)
    const double2 w32 = tw1024[32];
    double2 wk = tw1024[lane];
#endif
#pragma unroll
    for (int i = 0; i < NI; ++i) {
#if MXB_XW_TWREC
        if (i % 4 == 0) { if (i) wk = tw1024[lane + 32 * i]; }
        else wk = cmul(wk, w32);
#endif
#pragma unroll
        for (int ln = 0; ln < 2; ++ln) {
            const int kx = lane + 32 * i;
            if (kx < XHX) {
                const double2 zk = Wc[ln * XM + (kx & (XM - 1))];
                const double2 zm = Wc[ln * XM + ((XM - kx) & (XM - 1))];
                // E = (Zk + conj Zm)/2, O = (Zk - conj Zm)/(2i), X = E + W^k O
                const double2 E = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
                const double2 Od = make_double2(0.5 * (zk.y + zm.y), -0.5 * (zk.x - zm.x));
#if MXB_XW_TWREC
                xo[ln][i] = cadd(E, cmul(wk, Od));
#else
                xo[ln][i] = cadd(E, cmul(tw1024[kx], Od));
#endif
            }
        }
    }
    __syncthreads();   // every warp is done with its tile: stage the output pair
#pragma unroll
    for (int ln = 0; ln < 2; ++ln)
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            const int kx = lane + 32 * i;
            if (kx < XHX) W[PM ? (kx * 2 + ln) * 3 + c : (ln * XHX + kx) * 3 + c] = xo[ln][i];
        }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        if (PM) {
            // out[kx][row][c]: the pair's 96 bytes per plane, as TMA boxes of 256 planes
            const int x = (int)(row0 * 6);
            tma_store_2d(&map_main, x, 0, W);
            tma_store_2d(&map_main, x, 256, W + 256 * 6);
            tma_store_2d(&map_tail, x, 512, W + 512 * 6);
        } else {
            // out[row][kx][c]: two contiguous rows of XHX * 48 bytes
            bulk_s2g(out + (row0 * CHP) * 3, W, XHX * 48);
            bulk_s2g(out + ((row0 + 1) * CHP) * 3, W + XHX * 3, XHX * 48);
        }
        bulk_commit();
#if MXB_XW_EXIT_READ
        // the CTA may exit once the store has read its shared memory; the
        // global writes complete with the grid (the CTA slot is not held for them)
        bulk_wait_read();
#else
        bulk_wait_all();
#endif
    }
}

template <bool PM>
__global__ void __launch_bounds__(96, 4)
k_c2r_w(const double2* __restrict__ X, int CHP, long long BLKE, double* __restrict__ out, long long cstride,
        int pitch, const double2* __restrict__ tw512, const double2* __restrict__ tw1024,
        const int* __restrict__ halt, const __grid_constant__ CUtensorMap map_main,
        const __grid_constant__ CUtensorMap map_tail, int pfd) {
    if (halt && *halt) return;
    // the input pair ([kx][line][c] by TMA boxes, or [line][kx][c] by two bulk
    // rows), then 3 x 1024 transpose tiles
    extern __shared__ __align__(128) double2 S[];
    __shared__ alignas(8) unsigned long long mbar;
    const int c = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long row0 = 2LL * blockIdx.x;
    if (threadIdx.x == 0) {
        mbar_init(&mbar);
        if (PM) {
            mbar_expect(&mbar, XHX * 96);
            const int x = (int)(row0 * 6);
            tma_load_2d(S, &map_main, x, 0, &mbar);
            tma_load_2d(S + 256 * 6, &map_main, x, 256, &mbar);
            tma_load_2d(S + 512 * 6, &map_tail, x, 512, &mbar);
            if (pfd && blockIdx.x + pfd < gridDim.x) {   // the spectra slice pfd CTAs ahead into L2
                const int xn = (int)((row0 + 2LL * pfd) * 6);
                tma_prefetch_2d(&map_main, xn, 0);
                tma_prefetch_2d(&map_main, xn, 256);
                tma_prefetch_2d(&map_tail, xn, 512);
            }
        } else {
            mbar_expect(&mbar, 2 * XHX * 48);
            bulk_g2s_tx(S, X + row0 * CHP * 3, XHX * 48, &mbar);
            bulk_g2s_tx(S + XHX * 3, X + (row0 + 1) * CHP * 3, XHX * 48, &mbar);
        }
    }
    __syncthreads();   // mbarrier initialised before anyone polls it
#if MXB_XW_TWPRE
    // the untangling twiddles do not depend on the spectra: load them while the
    // TMA boxes are in flight
    double2 twp[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) twp[m] = __ldg(tw1024 + lane + 32 * m);
#endif
    mbar_wait(&mbar, 0);
    double2 a[16], b[16], v[32];
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        const int k = lane + 32 * m;
#if MXB_XW_TWPRE
        const double2 w = twp[m];
#else
        const double2 w = tw1024[k];
#endif
#pragma unroll
        for (int ln = 0; ln < 2; ++ln) {
            const double2 xk = S[PM ? (k * 2 + ln) * 3 + c : (ln * XHX + k) * 3 + c];
            const double2 xm = S[PM ? ((XM - k) * 2 + ln) * 3 + c : (ln * XHX + (XM - k)) * 3 + c];
            // Z = (Xk + conj Xm) + i (Xk - conj Xm) W^-k
            const double2 A = make_double2(xk.x + xm.x, xk.y - xm.y);
            const double2 Bm = make_double2(xk.x - xm.x, xk.y + xm.y);
            const double2 B = cmul(Bm, make_double2(w.x, -w.y));
            const double2 z = make_double2(A.x - B.y, A.y + B.x);
            if (ln == 0) a[m] = z; else b[m] = z;
        }
    }
    __syncthreads();   // S becomes the transpose tiles
    fw::fft512x2<1>(a, b, v, S + c * 1024, lane, tw512);
    const int line = lane >> 4, k1 = lane & 15;
    double2* dst = reinterpret_cast<double2*>(out + c * cstride + (row0 + line) * pitch);
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) dst[k1 + 16 * k2] = v[fw::p32(k2)];   // n < 256: x[2n], x[2n+1]
}

// -1 when the shape is not covered (the radix-16 kernels take it)
int warp_rows(bool fwd, int M, const double* in_r, double2* X, double* out_r, long long cstride, int pitch,
              int nhalf, int CH, int CHP, long long BLKE, long long nrows, const double2* twM,
              const double2* tw2M, cudaStream_t st, const int* halt) {
    const char* xe = getenv("MXB_XWARP");
    const bool on = !(xe && xe[0] == '0');
    if (!on || M != XM || nhalf != XM / 2 || (nrows & 1) || pitch != XM) return -1;
    const bool pm = CH == 1;
    // r2c: L2 prefetch of the input rows pfd CTAs ahead (MXB_XW_PFD, read per launch;
    // 0 = off); c2r: of its spectrum slice by tensor prefetch (MXB_XW_PFD_C2R, off:
    // measured 70% slower)
    const char* pe = getenv(fwd ? "MXB_XW_PFD" : "MXB_XW_PFD_C2R");
    const int pfd = pe ? atoi(pe) : (fwd ? MXB_XW_PFD_DEFAULT : 0);
    if (!pm && CH < XHX) return -1;   // row-major only for a single rank
    const unsigned grid = (unsigned)(nrows / 2);
    const size_t smem_r2c = (size_t)2 * XHX * 3 * sizeof(double2);   // >= the tiles
    const size_t smem_c2r = (size_t)2 * XHX * 3 * sizeof(double2);   // >= the tiles
    static bool attrs = false;
    if (!attrs) {
        MXB_CUDA(cudaFuncSetAttribute(k_r2c_w<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_r2c));
        MXB_CUDA(cudaFuncSetAttribute(k_r2c_w<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_r2c));
        MXB_CUDA(cudaFuncSetAttribute(k_c2r_w<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_c2r));
        MXB_CUDA(cudaFuncSetAttribute(k_c2r_w<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_c2r));
        for (const void* f : {(const void*)k_r2c_w<true>, (const void*)k_r2c_w<false>, (const void*)k_c2r_w<true>,
                              (const void*)k_c2r_w<false>})
            MXB_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        attrs = true;
    }
    // plane-major spectra as a 2-D float64 tensor: one row of nrows * 6 values
    // per kx plane; boxes of {2 rows x 3 components x 2, 256 | 1 planes}
    CUtensorMap mm{}, mt{};
    if (pm) {
        const unsigned long long inner = (unsigned long long)nrows * 6, pitch_b = (unsigned long long)BLKE * 16;
        if (make_map_2d_f64(&mm, X, inner, XHX, pitch_b, 12, 256) || make_map_2d_f64(&mt, X, inner, XHX, pitch_b, 12, 1))
            return MXB_ECUDA;
    }
    if (fwd) {
        if (pm) k_r2c_w<true><<<grid, 96, smem_r2c, st>>>(in_r, cstride, pitch, X, CHP, BLKE, twM, tw2M, halt, mm, mt, pfd);
        else k_r2c_w<false><<<grid, 96, smem_r2c, st>>>(in_r, cstride, pitch, X, CHP, BLKE, twM, tw2M, halt, mm, mt, pfd);
    } else {
        if (pm) k_c2r_w<true><<<grid, 96, smem_c2r, st>>>(X, CHP, BLKE, out_r, cstride, pitch, twM, tw2M, halt, mm, mt, pfd);
        else k_c2r_w<false><<<grid, 96, smem_c2r, st>>>(X, CHP, BLKE, out_r, cstride, pitch, twM, tw2M, halt, mm, mt, pfd);
    }
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

}  // namespace mxb
