// FNO demag surrogate inference on the GPU (the second .field backend,
// magnex/fno.py:228-447).
//
// Thin film (nz = 1), channels-first float64 fields (c, H, W) with H = ny,
// W = nx, as FnoModel.infer.  Per forward pass:
//   lift      v = lift_w . ((x - in_mean)/in_std) + lift_b           (fno.py:382-383)
//   4 blocks  v = act( spectral_conv(v) + (loc_w . v + loc_b) )     (fno.py:384-390)
//   proj      y = (proj_w . v + proj_b) * out_std + out_mean        (fno.py:391-392)
// spectral_conv keeps rows [0, m1) and [H-m1, H) of the half spectrum and
// columns [0, m2) (fno.py:228-255).  Only those 2*m1*m2 modes survive, so the
// transforms are truncated DFTs against exact twiddle tables instead of full
// FFTs: forward along x (W -> m2) then y (H -> 2 m1), the per-mode channel
// mix, inverse along y (2 m1 -> H), then the c2r along x fused with the 1x1
// bypass, bias and activation.  irfft2 semantics: scale 1/(H W), the
// imaginary part of the kx = 0 column is dropped, kx >= 1 counted twice
// (kx < m2 <= W/2, so no Nyquist column is ever kept).
#include <math.h>
#include <string.h>

#include <vector>

#include "common.cuh"
#include "fft_generic.cuh"

namespace mxb {

struct FnoDev {
    int dev = 0, w = 0, m1 = 0, m2 = 0, H = 0, W = 0, act = 0;
    cudaStream_t st = nullptr;
    double* params = nullptr;   // everything below points into it
    const double *lift_w, *lift_b, *loc_w[4], *loc_b[4], *proj_w, *proj_b, *norm;
    const double2 *wpos[4], *wneg[4];
    double2* ex = nullptr;   // [m2][W]   exp(-2 pi i kx x / W)
    double2* ey = nullptr;   // [2 m1][H] exp(-2 pi i ky y / H), ky = r < m1 ? r : H - 2 m1 + r
    double *v0 = nullptr, *v1 = nullptr;   // (w, H, W)
    double2 *A = nullptr, *Xf = nullptr, *Yf = nullptr, *C = nullptr;
    double* io = nullptr;    // 2 x (3, H, W) staging for host calls
};

static size_t fno_param_count(int w, int m1, int m2) {
    return (size_t)3 * w + w + 4 * ((size_t)4 * w * w * m1 * m2 + (size_t)w * w + w) + 3 * (size_t)w + 3 + 12;
}

__device__ __forceinline__ double act_fn(double x, int act) {
    if (act == 1) return x > 0.0 ? x : 0.0;
    return 0.5 * x * (1.0 + erf(x / 1.4142135623730951));
}

__global__ void k_fno_lift(const double* __restrict__ x, double* __restrict__ v, const double* __restrict__ lw,
                           const double* __restrict__ lb, const double* __restrict__ norm, int w, long long HW) {
    const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (p >= HW) return;
    double xn[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) xn[c] = (x[c * HW + p] - norm[c]) / norm[3 + c];
    for (int o = 0; o < w; ++o) {
        double s = lw[o * 3] * xn[0];
        s = s + lw[o * 3 + 1] * xn[1];
        s = s + lw[o * 3 + 2] * xn[2];
        v[o * HW + p] = s + lb[o];
    }
}

// A[c][y][kx] = sum_x v[c][y][x] ex[kx][x]
__global__ void k_fno_dft_x(const double* __restrict__ v, double2* __restrict__ A, const double2* __restrict__ ex,
                            int rows, int W, int m2) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= (long long)rows * m2) return;
    const int kx = (int)(t % m2);
    const long long row = t / m2;
    const double* vr = v + row * W;
    const double2* e = ex + (long long)kx * W;
    double re = 0.0, im = 0.0;
    for (int x = 0; x < W; ++x) {
        const double a = __ldg(vr + x);
        const double2 z = __ldg(e + x);
        re = fma(a, z.x, re);
        im = fma(a, z.y, im);
    }
    A[t] = make_double2(re, im);
}

// Blocked forms of the two large passes (the per-output loops above re-read the
// twiddle table and the input row m2 / w times from L2; at 2048^2 they were
// ~95% of the forward pass):
//   k_fno_dft_x_w: one warp per row, lanes over x, all m2 <= 12 outputs
//   accumulated in registers against table chunks staged in shared memory,
//   warp-shuffle reduction at the end;
//   k_fno_block_out_t: one thread per x of a row, the w <= MAXW input channels
//   of that cell in registers, C[:, y, :], the bypass weights and a table chunk
//   in shared memory, all w outputs from one pass.
constexpr int kFnoChunk = 128;   // x values per staged table chunk

template <int MAXM2>
__global__ void __launch_bounds__(256) k_fno_dft_x_w(const double* __restrict__ v, double2* __restrict__ A,
                                                     const double2* __restrict__ ex, int rows, int W, int m2) {
    __shared__ double2 es[MAXM2][kFnoChunk];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long row = (long long)blockIdx.x * 8 + warp;
    const double* vr = v + row * W;
    double2 acc[MAXM2];
#pragma unroll
    for (int k = 0; k < MAXM2; ++k) acc[k] = make_double2(0.0, 0.0);
    for (int x0 = 0; x0 < W; x0 += kFnoChunk) {
        const int n = min(kFnoChunk, W - x0);
        __syncthreads();
        for (int i = threadIdx.x; i < m2 * kFnoChunk; i += 256) {
            const int k = i / kFnoChunk, x = i - k * kFnoChunk;
            if (x < n) es[k][x] = __ldg(ex + (long long)k * W + x0 + x);
        }
        __syncthreads();
        if (row < rows) {
            for (int x = lane; x < n; x += 32) {
                const double a = __ldg(vr + x0 + x);
#pragma unroll
                for (int k = 0; k < MAXM2; ++k)
                    if (k < m2) {
                        acc[k].x = fma(a, es[k][x].x, acc[k].x);
                        acc[k].y = fma(a, es[k][x].y, acc[k].y);
                    }
            }
        }
    }
    if (row >= rows) return;
#pragma unroll
    for (int k = 0; k < MAXM2; ++k) {
        if (k >= m2) break;
        double re = acc[k].x, im = acc[k].y;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            re += __shfl_xor_sync(0xffffffffu, re, o);
            im += __shfl_xor_sync(0xffffffffu, im, o);
        }
        if (lane == 0) A[row * m2 + k] = make_double2(re, im);
    }
}

template <int MAXW, int MAXM2>
__global__ void __launch_bounds__(kFnoChunk) k_fno_block_out_t(const double2* __restrict__ C, const double* __restrict__ vin,
                                                               double* __restrict__ vout, const double2* __restrict__ ex,
                                                               const double* __restrict__ lw, const double* __restrict__ lb,
                                                               int w, int H, int W, int m2, int act, double scale) {
    __shared__ double2 cs[MAXW][MAXM2];
    __shared__ double2 es[MAXM2][kFnoChunk];
    __shared__ double ws[MAXW][MAXW + 1];
    __shared__ double bs[MAXW];
    const long long HW = (long long)H * W;
    const int y = blockIdx.y, x0 = blockIdx.x * kFnoChunk, x = x0 + threadIdx.x;
    for (int i = threadIdx.x; i < w * m2; i += kFnoChunk) {
        const int o = i / m2, k = i - o * m2;
        cs[o][k] = C[((long long)o * H + y) * m2 + k];
    }
    for (int i = threadIdx.x; i < m2 * kFnoChunk; i += kFnoChunk) {
        const int k = i / kFnoChunk, xx = i - k * kFnoChunk;
        if (x0 + xx < W) es[k][xx] = __ldg(ex + (long long)k * W + x0 + xx);
    }
    if (lw) {
        for (int i = threadIdx.x; i < w * w; i += kFnoChunk) ws[i / w][i % w] = lw[i];
        for (int i = threadIdx.x; i < w; i += kFnoChunk) bs[i] = lb[i];
    }
    __syncthreads();
    if (x >= W) return;
    const long long p = (long long)y * W + x;
    double vi[MAXW];
#pragma unroll
    for (int i = 0; i < MAXW; ++i) vi[i] = (lw && i < w) ? __ldg(vin + i * HW + p) : 0.0;
    for (int o = 0; o < w; ++o) {
        double s = cs[o][0].x;
#pragma unroll
        for (int k = 1; k < MAXM2; ++k)
            if (k < m2) {
                const double2 z = cs[o][k], e = es[k][threadIdx.x];
                s += 2.0 * (z.x * e.x + z.y * e.y);
            }
        s *= scale;
        double r = s;
        if (lw) {
            double l = 0.0;
#pragma unroll
            for (int i = 0; i < MAXW; ++i)
                if (i < w) l = fma(ws[o][i], vi[i], l);
            r = s + (l + bs[o]);
        }
        if (act >= 0) r = act_fn(r, act);
        vout[o * HW + p] = r;
    }
}

// X[c][r][kx] = sum_y A[c][y][kx] ey[r][y]
__global__ void k_fno_dft_y(const double2* __restrict__ A, double2* __restrict__ X, const double2* __restrict__ ey,
                            int w, int H, int m1, int m2) {
    const int R = 2 * m1;
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= (long long)w * R * m2) return;
    const int kx = (int)(t % m2);
    const int r = (int)((t / m2) % R);
    const int c = (int)(t / ((long long)m2 * R));
    const double2* a = A + (long long)c * H * m2 + kx;
    const double2* e = ey + (long long)r * H;
    double2 s = make_double2(0.0, 0.0);
    for (int y = 0; y < H; ++y) {
        const double2 p = __ldg(a + (long long)y * m2), q = __ldg(e + y);
        s.x = fma(p.x, q.x, fma(-p.y, q.y, s.x));
        s.y = fma(p.x, q.y, fma(p.y, q.x, s.y));
    }
    X[t] = s;
}

// Y[o][r][kx] = sum_i X[i][r][kx] Wt[i][o][r mod m1][kx], Wt = pos for r < m1, neg otherwise
__global__ void k_fno_mix(const double2* __restrict__ X, double2* __restrict__ Y, const double2* __restrict__ wp,
                          const double2* __restrict__ wn, int w, int m1, int m2) {
    const int R = 2 * m1;
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= (long long)w * R * m2) return;
    const int kx = (int)(t % m2);
    const int r = (int)((t / m2) % R);
    const int o = (int)(t / ((long long)m2 * R));
    const double2* wt = r < m1 ? wp : wn;
    const int rr = r < m1 ? r : r - m1;
    double2 s = make_double2(0.0, 0.0);
    for (int i = 0; i < w; ++i) {
        const double2 p = X[((long long)i * R + r) * m2 + kx];
        const double2 q = __ldg(wt + (((long long)i * w + o) * m1 + rr) * m2 + kx);
        s = cadd(s, cmul(p, q));
    }
    Y[t] = s;
}

// C[o][y][kx] = sum_r Y[o][r][kx] conj(ey[r][y])
__global__ void k_fno_idft_y(const double2* __restrict__ Y, double2* __restrict__ C, const double2* __restrict__ ey,
                             int w, int H, int m1, int m2) {
    const int R = 2 * m1;
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= (long long)w * H * m2) return;
    const int kx = (int)(t % m2);
    const int y = (int)((t / m2) % H);
    const int o = (int)(t / ((long long)m2 * H));
    double2 s = make_double2(0.0, 0.0);
    for (int r = 0; r < R; ++r) {
        const double2 p = Y[((long long)o * R + r) * m2 + kx];
        const double2 q = __ldg(ey + (long long)r * H + y);
        // p * conj(q)
        s.x = fma(p.x, q.x, fma(p.y, q.y, s.x));
        s.y = fma(p.y, q.x, fma(-p.x, q.y, s.y));
    }
    C[t] = s;
}

// vout[o][p] = act( c2r(C)[o][p] + (sum_i lw[o][i] vin[i][p] + lb[o]) ); act < 0: none
__global__ void k_fno_block_out(const double2* __restrict__ C, const double* __restrict__ vin,
                                double* __restrict__ vout, const double2* __restrict__ ex,
                                const double* __restrict__ lw, const double* __restrict__ lb, int w, int H, int W,
                                int m2, int act, double scale) {
    const long long HW = (long long)H * W;
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= (long long)w * HW) return;
    const long long p = t % HW;
    const int o = (int)(t / HW);
    const int y = (int)(p / W), x = (int)(p - (long long)y * W);
    const double2* c = C + ((long long)o * H + y) * m2;
    double s = c[0].x;
    for (int kx = 1; kx < m2; ++kx) {
        const double2 z = c[kx], e = __ldg(ex + (long long)kx * W + x);
        // 2 Re(z * conj(e))
        s += 2.0 * (z.x * e.x + z.y * e.y);
    }
    s *= scale;
    double r = s;
    if (lw) {   // bypass: s + (loc_w . v + loc_b), the reference's association
        double l = 0.0;
        for (int i = 0; i < w; ++i) l = fma(lw[o * w + i], vin[i * HW + p], l);
        r = s + (l + lb[o]);
    }
    if (act >= 0) r = act_fn(r, act);
    vout[t] = r;
}

__global__ void k_fno_proj(const double* __restrict__ v, double* __restrict__ y, const double* __restrict__ pw,
                           const double* __restrict__ pb, const double* __restrict__ norm, int w, long long HW) {
    const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (p >= HW) return;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        double s = 0.0;
        for (int o = 0; o < w; ++o) s = fma(pw[c * w + o], v[o * HW + p], s);
        y[c * HW + p] = (s + pb[c]) * norm[9 + c] + norm[6 + c];
    }
}

static unsigned nblk(long long n, int t) { return (unsigned)((n + t - 1) / t); }

static int fno_tables(FnoDev& f) {
    std::vector<double2> ex((size_t)f.m2 * f.W), ey((size_t)2 * f.m1 * f.H);
    const long double tau = 6.283185307179586476925286766559005768L;
    for (int k = 0; k < f.m2; ++k)
        for (int x = 0; x < f.W; ++x) {
            const long double a = -tau * (long double)(((long long)k * x) % f.W) / f.W;
            ex[(size_t)k * f.W + x] = make_double2((double)cosl(a), (double)sinl(a));
        }
    for (int r = 0; r < 2 * f.m1; ++r) {
        const int ky = r < f.m1 ? r : f.H - 2 * f.m1 + r;
        for (int y = 0; y < f.H; ++y) {
            const long double a = -tau * (long double)(((long long)ky * y) % f.H) / f.H;
            ey[(size_t)r * f.H + y] = make_double2((double)cosl(a), (double)sinl(a));
        }
    }
    MXB_CUDA(cudaMalloc(&f.ex, ex.size() * sizeof(double2)));
    MXB_CUDA(cudaMalloc(&f.ey, ey.size() * sizeof(double2)));
    MXB_CUDA(cudaMemcpy(f.ex, ex.data(), ex.size() * sizeof(double2), cudaMemcpyHostToDevice));
    MXB_CUDA(cudaMemcpy(f.ey, ey.data(), ey.size() * sizeof(double2), cudaMemcpyHostToDevice));
    return MXB_OK;
}

static int fno_buffers(FnoDev& f) {
    const size_t HW = (size_t)f.H * f.W;
    MXB_CUDA(cudaMalloc(&f.v0, (size_t)f.w * HW * sizeof(double)));
    MXB_CUDA(cudaMalloc(&f.v1, (size_t)f.w * HW * sizeof(double)));
    MXB_CUDA(cudaMalloc(&f.A, (size_t)f.w * f.H * f.m2 * sizeof(double2)));
    MXB_CUDA(cudaMalloc(&f.C, (size_t)f.w * f.H * f.m2 * sizeof(double2)));
    MXB_CUDA(cudaMalloc(&f.Xf, (size_t)f.w * 2 * f.m1 * f.m2 * sizeof(double2)));
    MXB_CUDA(cudaMalloc(&f.Yf, (size_t)f.w * 2 * f.m1 * f.m2 * sizeof(double2)));
    MXB_CUDA(cudaMalloc(&f.io, 2 * 3 * HW * sizeof(double)));
    return MXB_OK;
}

static void fno_free(FnoDev& f) {
    cudaSetDevice(f.dev);
    for (void* p : {(void*)f.params, (void*)f.ex, (void*)f.ey, (void*)f.v0, (void*)f.v1, (void*)f.A, (void*)f.C,
                    (void*)f.Xf, (void*)f.Yf, (void*)f.io})
        if (p) cudaFree(p);
    if (f.st) cudaStreamDestroy(f.st);
}

// spectral conv of vin (c = w channels) with block k's filters, added to the
// bypass of vin, into vout.  With lw == nullptr: the bare spectral_conv.
static int fno_block(FnoDev& f, const double* vin, double* vout, const double2* wp, const double2* wn,
                     const double* lw, const double* lb, int act) {
    const int T = 256, w = f.w, R = 2 * f.m1;
    const long long HW = (long long)f.H * f.W;
    if (f.m2 <= 12)
        k_fno_dft_x_w<12><<<nblk((long long)w * f.H, 8), 256, 0, f.st>>>(vin, f.A, f.ex, w * f.H, f.W, f.m2);
    else
        k_fno_dft_x<<<nblk((long long)w * f.H * f.m2, T), T, 0, f.st>>>(vin, f.A, f.ex, w * f.H, f.W, f.m2);
    k_fno_dft_y<<<nblk((long long)w * R * f.m2, T), T, 0, f.st>>>(f.A, f.Xf, f.ey, w, f.H, f.m1, f.m2);
    k_fno_mix<<<nblk((long long)w * R * f.m2, T), T, 0, f.st>>>(f.Xf, f.Yf, wp, wn, w, f.m1, f.m2);
    k_fno_idft_y<<<nblk((long long)w * f.H * f.m2, T), T, 0, f.st>>>(f.Yf, f.C, f.ey, w, f.H, f.m1, f.m2);
    if (w <= 32 && f.m2 <= 12) {
        const dim3 grid((unsigned)((f.W + kFnoChunk - 1) / kFnoChunk), (unsigned)f.H);
        k_fno_block_out_t<32, 12><<<grid, kFnoChunk, 0, f.st>>>(f.C, vin, vout, f.ex, lw, lb, w, f.H, f.W, f.m2,
                                                               act, 1.0 / ((double)f.H * f.W));
    } else {
        k_fno_block_out<<<nblk((long long)w * HW, T), T, 0, f.st>>>(f.C, vin, vout, f.ex, lw, lb, w, f.H, f.W,
                                                                    f.m2, act, 1.0 / ((double)f.H * f.W));
    }
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

static int fno_forward(FnoDev& f, const double* x, double* y) {
    const int T = 256;
    const long long HW = (long long)f.H * f.W;
    k_fno_lift<<<nblk(HW, T), T, 0, f.st>>>(x, f.v0, f.lift_w, f.lift_b, f.norm, f.w, HW);
    MXB_LAUNCH_CHECK();
    double *a = f.v0, *b = f.v1;
    for (int k = 0; k < 4; ++k) {
        int rc = fno_block(f, a, b, f.wpos[k], f.wneg[k], f.loc_w[k], f.loc_b[k], k < 3 ? f.act : -1);
        if (rc) return rc;
        double* t = a;
        a = b;
        b = t;
    }
    k_fno_proj<<<nblk(HW, T), T, 0, f.st>>>(a, y, f.proj_w, f.proj_b, f.norm, f.w, HW);
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

}  // namespace mxb

using namespace mxb;

struct mxb_fno {
    FnoDev f;
};

extern "C" {

int mxb_fno_create(int device, int width, int m1, int m2, int ny, int nx, int activation, const double* params,
                   mxb_fno** out) {
    if (!out || !params) { set_error("null argument"); return MXB_EINVAL; }
    *out = nullptr;
    if (width < 1 || m1 < 1 || m2 < 1) { set_error("FNO width and modes must be positive"); return MXB_EINVAL; }
    if (activation != 0 && activation != 1) { set_error("unknown activation code"); return MXB_EINVAL; }
    if (ny < 2 * m1 || nx < 2 * m2) {
        set_error("grid has insufficient spectral extent for the modes");
        return MXB_EINVAL;
    }
    auto* h = new mxb_fno();
    FnoDev& f = h->f;
    f.dev = device;
    f.w = width; f.m1 = m1; f.m2 = m2; f.H = ny; f.W = nx; f.act = activation;
    int rc = MXB_OK;
    auto fail = [&](int r) { fno_free(f); delete h; return r; };
    if (cudaSetDevice(device) != cudaSuccess) { set_error("bad device"); return fail(MXB_ECUDA); }
    if (cudaStreamCreateWithFlags(&f.st, cudaStreamNonBlocking) != cudaSuccess) { set_error("stream"); return fail(MXB_ECUDA); }
    const size_t n = fno_param_count(width, m1, m2);
    if (cudaMalloc(&f.params, n * sizeof(double)) != cudaSuccess) { set_error("out of device memory"); return fail(MXB_ECUDA); }
    if (cudaMemcpy(f.params, params, n * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) {
        set_error("parameter upload failed");
        return fail(MXB_ECUDA);
    }
    const double* p = f.params;
    f.lift_w = p; p += 3 * width;
    f.lift_b = p; p += width;
    const size_t spec = (size_t)width * width * m1 * m2;
    for (int k = 0; k < 4; ++k) {
        f.wpos[k] = reinterpret_cast<const double2*>(p); p += 2 * spec;
        f.wneg[k] = reinterpret_cast<const double2*>(p); p += 2 * spec;
        f.loc_w[k] = p; p += (size_t)width * width;
        f.loc_b[k] = p; p += width;
    }
    f.proj_w = p; p += 3 * width;
    f.proj_b = p; p += 3;
    f.norm = p;
    if ((rc = fno_tables(f)) || (rc = fno_buffers(f))) return fail(rc);
    *out = h;
    return MXB_OK;
}

void mxb_fno_destroy(mxb_fno* h) {
    if (!h) return;
    fno_free(h->f);
    delete h;
}

}  // extern "C"

namespace mxb {
// the forward pass on another stream (the solver's: the surrogate runs inside
// the captured step of mxb_run, api.cu demag_into)
int fno_forward_on(mxb_fno* h, const double* x, double* y, cudaStream_t st, int* H, int* W) {
    if (!h) { set_error("null argument"); return MXB_EINVAL; }
    if (H) *H = h->f.H;
    if (W) *W = h->f.W;
    if (!x || !y) return MXB_OK;
    cudaStream_t own = h->f.st;
    h->f.st = st;
    const int rc = fno_forward(h->f, x, y);
    h->f.st = own;
    return rc;
}
}  // namespace mxb

extern "C" {

int mxb_fno_infer_dev(mxb_fno* h, const double* x, double* y) {
    if (!h || !x || !y) { set_error("null argument"); return MXB_EINVAL; }
    cudaSetDevice(h->f.dev);
    return fno_forward(h->f, x, y);
}

int mxb_fno_infer(mxb_fno* h, const double* x_host, double* y_host) {
    if (!h || !x_host || !y_host) { set_error("null argument"); return MXB_EINVAL; }
    FnoDev& f = h->f;
    cudaSetDevice(f.dev);
    const size_t b = (size_t)3 * f.H * f.W * sizeof(double);
    MXB_CUDA(cudaMemcpyAsync(f.io, x_host, b, cudaMemcpyHostToDevice, f.st));
    int rc = fno_forward(f, f.io, f.io + 3 * (size_t)f.H * f.W);
    if (rc) return rc;
    MXB_CUDA(cudaMemcpyAsync(y_host, f.io + 3 * (size_t)f.H * f.W, b, cudaMemcpyDeviceToHost, f.st));
    MXB_CUDA(cudaStreamSynchronize(f.st));
    return MXB_OK;
}

int mxb_fno_spectral_conv(int device, int channels, int ny, int nx, int m1, int m2, const double* w_pos,
                          const double* w_neg, const double* x_host, double* y_host) {
    if (!w_pos || !w_neg || !x_host || !y_host) { set_error("null argument"); return MXB_EINVAL; }
    if (channels < 1 || m1 < 1 || m2 < 1) { set_error("channels and modes must be positive"); return MXB_EINVAL; }
    if (ny < 2 * m1 || nx < 2 * m2) { set_error("grid has insufficient spectral extent for the modes"); return MXB_EINVAL; }
    FnoDev f;
    f.dev = device;
    f.w = channels; f.m1 = m1; f.m2 = m2; f.H = ny; f.W = nx; f.act = -1;
    int rc = MXB_OK;
    cudaSetDevice(device);
    const size_t spec = (size_t)channels * channels * m1 * m2;
    const size_t HW = (size_t)ny * nx;
    do {
        if (cudaStreamCreateWithFlags(&f.st, cudaStreamNonBlocking) != cudaSuccess) {
            rc = cuda_fail(cudaGetLastError(), "stream", __FILE__, __LINE__);
            break;
        }
        if (cudaMalloc(&f.params, 4 * spec * sizeof(double)) != cudaSuccess) {
            rc = cuda_fail(cudaGetLastError(), "cudaMalloc", __FILE__, __LINE__);
            break;
        }
        cudaMemcpy(f.params, w_pos, 2 * spec * sizeof(double), cudaMemcpyHostToDevice);
        cudaMemcpy(f.params + 2 * spec, w_neg, 2 * spec * sizeof(double), cudaMemcpyHostToDevice);
        if ((rc = fno_tables(f)) || (rc = fno_buffers(f))) break;
        cudaMemcpyAsync(f.v0, x_host, (size_t)channels * HW * sizeof(double), cudaMemcpyHostToDevice, f.st);
        rc = fno_block(f, f.v0, f.v1, reinterpret_cast<const double2*>(f.params),
                       reinterpret_cast<const double2*>(f.params + 2 * spec), nullptr, nullptr, -1);
        if (rc) break;
        cudaMemcpyAsync(y_host, f.v1, (size_t)channels * HW * sizeof(double), cudaMemcpyDeviceToHost, f.st);
        if (cudaStreamSynchronize(f.st) != cudaSuccess) { rc = cuda_fail(cudaGetLastError(), "spectral_conv", __FILE__, __LINE__); break; }
    } while (false);
    fno_free(f);
    return rc;
}

}  // extern "C"
