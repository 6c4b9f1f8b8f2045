// Long y lines (py = 2048 / 4096, e.g. the 2048 x 2048 x 64 film), one rank or
// a z slab (each rank its kx chunk, rows read from the all-to-all blocks).
//
// The 5-pass path keeps the spectra row-major, X[z][y][kx][c]: a y column is
// 16 B every CHP*48 B (98 KB apart at hx = 2049) and two 4096-point lines per
// CTA need 139 KB of shared memory, so the column passes ran at 18% of HBM.
// Here the x passes write the plane-major layout of the plane pipeline,
// XR[kx][z][y][c], so a y line of the three components is one contiguous row:
//   y forward   k_yrow<L,-1>: row (kx, z) of ny x 48 B -> X2[kx][z][ky][c] (py x 48 B)
//   z fused     k_fused_fast<pz, 4> over X2 with ky as the contiguous lane
//               (NK consecutive ky per tile) and the quarter kernel
//               Kp[kx][ky'][kz'][6] (ky, kz folded; parity signs of XY/XZ/YZ)
//   y inverse   k_yrow<L,+1>: X2 row (py x 48 B) -> XR row, ny kept
// One CTA per row: the row is staged with bulk copies into the shared
// buffer, transformed by the radix-16 CTA core (fft_fast.cuh, the three
// components as three lines), written back in natural order and stored with
// one bulk store.
#include <stdlib.h>

#include "demag.cuh"
#include "fft_fast.cuh"
#include "tma.cuh"

namespace mxb {

using namespace ff;

namespace {
template <int L> struct YRowCfg {
    static constexpr int R = 16;
    static constexpr int TPL = L / R;
    static constexpr int T = 3 * TPL;
    static constexpr int XE = smem_elems<L, R, 3>();   // exchange buffer, >= 3 L
};
constexpr unsigned kChunk = 32768;   // bytes per bulk copy
}  // namespace

// the XR side of a row (kx, z) = blockIdx.x = kx * nz + z: contiguous rows on
// one rank; on a z slab the all-to-all receive blocks [g][kx][z_l][y][3]
// (row z of plane kx in block z / nzl, nzl a power of two; zjump = block
// stride / nzl), as the plane pipeline reads them
struct YRowSlab {
    int nz, nzl;
    long long zjump;
    __device__ long long row(long long r, int n) const {
        const long long kx = r / nz;
        const int z = (int)(r - kx * nz), zl = nzl == nz ? z : (z & (nzl - 1));
        return (long long)(z - zl) * zjump + (kx * nzl + zl) * (long long)n * 3;
    }
};

template <int L, int DIR>
__global__ void __launch_bounds__(YRowCfg<L>::T, 1)
k_yrow(const double2* __restrict__ in, double2* __restrict__ out, int n_in, int n_out,
       const double2* __restrict__ tw, const int* __restrict__ halt, YRowSlab sl) {
    if (halt && *halt) return;
    constexpr int R = YRowCfg<L>::R, TPL = YRowCfg<L>::TPL;
    extern __shared__ __align__(128) double2 X[];
    __shared__ alignas(8) unsigned long long mbar;
    const long long row = blockIdx.x;
    // forward: XR (slab rows) -> X2 (local rows); inverse: X2 -> XR
    const double2* src = in + (DIR < 0 ? sl.row(row, n_in) : row * (long long)n_in * 3);
    double2* dst = out + (DIR < 0 ? row * (long long)n_out * 3 : sl.row(row, n_out));
    const int b = threadIdx.x / TPL, t = threadIdx.x - b * TPL;
    if (threadIdx.x == 0) {
        mbar_init(&mbar);
        const unsigned bytes = (unsigned)n_in * 48u;
        mbar_expect(&mbar, bytes);
        for (unsigned o = 0; o < bytes; o += kChunk)
            bulk_g2s_tx(reinterpret_cast<char*>(X) + o, reinterpret_cast<const char*>(src) + o,
                        bytes - o < kChunk ? bytes - o : kChunk, &mbar);
    }
    __syncthreads();
    mbar_wait(&mbar, 0);
    double2 v[R];
#pragma unroll
    for (int m = 0; m < R; ++m) {
        const int e = t + m * TPL;
        v[m] = e < n_in ? X[e * 3 + b] : make_double2(0.0, 0.0);
    }
    fft_core<L, R, 3, false, DIR>(v, X, b, t, tw);   // opens with a barrier
    __syncthreads();
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const int e = out_elem<L, R>(t, i);
        if (e < n_out) X[e * 3 + b] = v[i];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned bytes = (unsigned)n_out * 48u;
        for (unsigned o = 0; o < bytes; o += kChunk)
            bulk_s2g(reinterpret_cast<char*>(dst) + o, reinterpret_cast<const char*>(X) + o,
                     bytes - o < kChunk ? bytes - o : kChunk);
        bulk_commit();
        bulk_wait_read();
    }
}

template <int L, int DIR>
static int yrow_launch(const double2* in, double2* out, int n_in, int n_out, long long rows, const double2* tw,
                       cudaStream_t st, const int* halt, YRowSlab sl) {
    const size_t smem = (size_t)YRowCfg<L>::XE * sizeof(double2);
    static bool attr = false;
    if (!attr) {
        MXB_CUDA(cudaFuncSetAttribute(k_yrow<L, DIR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    k_yrow<L, DIR><<<(unsigned)rows, YRowCfg<L>::T, smem, st>>>(in, out, n_in, n_out, tw, halt, sl);
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

bool longy_shape_ok(int py) { return py == 2048 || py == 4096; }

int longy_rows(int dir, int L, const double2* in, double2* out, int n_in, int n_out, long long rows,
               const double2* tw, cudaStream_t st, const int* halt, int nz, int nzl, long long gstride) {
    if (nzl <= 0) nzl = nz;
    if (nzl != nz && ((nzl & (nzl - 1)) || nz % nzl || gstride % nzl)) {
        set_error("long-y slab: the local planes must be a power of two dividing nz");
        return MXB_EINVAL;
    }
    const YRowSlab sl{nz, nzl, nzl != nz ? gstride / nzl : 0};
    if (L == 2048) return dir < 0 ? yrow_launch<2048, -1>(in, out, n_in, n_out, rows, tw, st, halt, sl)
                                  : yrow_launch<2048, 1>(in, out, n_in, n_out, rows, tw, st, halt, sl);
    if (L == 4096) return dir < 0 ? yrow_launch<4096, -1>(in, out, n_in, n_out, rows, tw, st, halt, sl)
                                  : yrow_launch<4096, 1>(in, out, n_in, n_out, rows, tw, st, halt, sl);
    set_error("no long-y row kernel for this length");
    return MXB_EINVAL;
}

// x forward of the long-y path: the row-major r2c ([z][y][hxp][3], contiguous
// rows) followed by this tiled transpose into the plane-major [kx][z][y][3]
// is faster at M = 2048 than the plane-major r2c, whose one row per CTA
// scatters 48-byte pieces over hx planes (9.1 + transpose vs 19.7 ms).
// Tile: 16 y x 32 kx of one z; reads 1.5 KB runs, writes 768-byte runs.
__global__ void __launch_bounds__(256) k_rm_to_pm(const double2* __restrict__ in, double2* __restrict__ out,
                                                  int ny, int nz, int hx, int hxp) {
    constexpr int TY = 16, TK = 32, W3 = TK * 3 + 1;
    __shared__ double2 tile[TY][W3];
    const int kx0 = blockIdx.x * TK, y0 = blockIdx.y * TY, z = blockIdx.z;
    for (int i = threadIdx.x; i < TY * TK * 3; i += 256) {
        const int yy = i / (TK * 3), q = i - yy * (TK * 3);
        const int y = y0 + yy, kx = kx0 + q / 3;
        if (y < ny && kx < hx) tile[yy][q] = in[(((long long)z * ny + y) * hxp + kx0) * 3 + q];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < TK * TY * 3; i += 256) {
        const int kk = i / (TY * 3), q = i - kk * (TY * 3);
        const int yy = q / 3, c = q - 3 * yy;
        const int kx = kx0 + kk, y = y0 + yy;
        if (y < ny && kx < hx) out[(((long long)kx * nz + z) * ny + y) * 3 + c] = tile[yy][kk * 3 + c];
    }
}

int longy_rm_to_pm(const double2* in, double2* out, int ny, int nz, int hx, int hxp, cudaStream_t st) {
    const dim3 grid((unsigned)((hx + 31) / 32), (unsigned)((ny + 15) / 16), (unsigned)nz);
    k_rm_to_pm<<<grid, 256, 0, st>>>(in, out, ny, nz, hx, hxp);
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

// K (complex full spectra [kz][ky][hxp][6], exactly real) -> Kp[kx][ky'][kz'][6],
// ky' <= py/2, kz' <= pz/2
__global__ void k_quarter_kx_major(const double2* __restrict__ K, double* __restrict__ Kp, int py, int pz,
                                   int hx, int hxp, int kx0) {
    const int Y2 = py / 2 + 1, Z2 = pz / 2 + 1;
    const long long tot = (long long)hx * Y2 * Z2 * 6;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
         i += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(i % 6);
        long long r = i / 6;
        const int kz = (int)(r % Z2);
        r /= Z2;
        const int ky = (int)(r % Y2);
        const int kx = (int)(r / Y2);
        Kp[i] = K[(((long long)kz * py + ky) * hxp + kx0 + kx) * 6 + c].x;
    }
}

int longy_quarter(const double2* K, double* Kp, int py, int pz, int hx, int hxp, cudaStream_t st, int kx0) {
    k_quarter_kx_major<<<148 * 8, 256, 0, st>>>(K, Kp, py, pz, hx, hxp, kx0);
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

}  // namespace mxb
