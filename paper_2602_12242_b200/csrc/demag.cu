// Zero-padded FFT demagnetising field (DemagKernel.field, demag.py:203-216).
//
// Pipeline for one evaluation (3 components, padded dims p = 2n or 1):
//   P1  x r2c of the nx real values of every (z,y) row, zero-padded to px,
//       keeping hx = px/2+1 bins -> X1[z][y][kx][c]      (component-interleaved)
//   P2  y c2c forward, ny non-zero rows -> py rows       -> X2[z][ky][kx][c]
//   P3  z c2c forward (nz non-zero) * symmetric 3x3 kernel multiply * z c2c
//       inverse, keeping the nz rows, in place in X2        (fused, one kernel)
//   P4  y c2c inverse, keeping the ny rows              -> X1
//   P5  x c2r of every row, keeping nx values, scaled by 1/(px py pz) -> H
// A thin film (nz = 1) fuses the y transform with the multiply instead.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "demag.cuh"
#include "fft_generic.cuh"

namespace mxb {

static std::vector<int> factorize(int L) {
    std::vector<int> r;
    while (L % 8 == 0 && L > 8) { r.push_back(8); L /= 8; }
    if (L == 8) { r.push_back(8); L = 1; }
    while (L % 4 == 0) { r.push_back(4); L /= 4; }
    while (L % 2 == 0) { r.push_back(2); L /= 2; }
    for (int f = 3; L > 1; f += 2)
        while (L % f == 0) { r.push_back(f); L /= f; }
    return r;
}

int make_plan(int L, int dev, Plan1D* p, double2** tw_owned) {
    p->L = L;
    std::vector<int> r = factorize(L);
    if (r.size() > 24) { set_error("FFT length has too many factors"); return MXB_EINVAL; }
    p->nst = (int)r.size();
    for (size_t i = 0; i < r.size(); ++i) p->radix[i] = r[i];
    std::vector<double2> h(L);
    for (int n = 0; n < L; ++n) {
        long double a = -2.0L * 3.14159265358979323846264338327950288L * (long double)n / (long double)L;
        h[n] = make_double2((double)cosl(a), (double)sinl(a));
    }
    double2* d = nullptr;
    MXB_CUDA(cudaMalloc(&d, sizeof(double2) * L));
    MXB_CUDA(cudaMemcpy(d, h.data(), sizeof(double2) * L, cudaMemcpyHostToDevice));
    p->tw = d;
    *tw_owned = d;
    return MXB_OK;
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------

// P1: rows of real input (line = (row, component), component fastest),
// zero-padded to L, forward FFT, first hx bins -> out[(row*hxp+kx)*nc + c].
__global__ void k_rows_r2c(const double* __restrict__ in, long long in_cstride, int in_pitch,
                           int n_in, double2* __restrict__ out, int hxp, int hx, int nc,
                           int ostride, int coff, int nrows, Plan1D p, int NL,
                           const int* __restrict__ halt) {
    if (halt && *halt) return;
    extern __shared__ double2 sm[];
    const int L = p.L, ld = L + 1;
    double2* a = sm;
    double2* b = sm + NL * ld;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const long long line0 = (long long)blockIdx.x * NL;
    const long long nlines = (long long)nrows * nc;
    for (int u = tid; u < NL * L; u += nthr) {
        const int l = u / L, e = u - l * L;
        const long long g = line0 + l;
        double v = 0.0;
        if (g < nlines && e < n_in) {
            const long long row = g / nc;
            const int c = (int)(g - row * nc);
            v = in[c * in_cstride + row * in_pitch + e];
        }
        a[l * ld + e] = make_double2(v, 0.0);
    }
    __syncthreads();
    double2* r = fft_lines<-1>(a, b, NL, p, tid, nthr);
    const int rows_here = NL / nc;
    const long long row0 = line0 / nc;
    for (int u = tid; u < rows_here * hx * nc; u += nthr) {
        const int rl = u / (hx * nc), q = u - rl * (hx * nc);
        const int kx = q / nc, c = q - kx * nc;
        const long long row = row0 + rl;
        if (row >= nrows) continue;
        out[(row * hxp + kx) * ostride + coff + c] = r[(rl * nc + c) * ld + kx];
    }
}

// P2/P4 (and the kernel-spectrum passes): strided complex lines.
// line g -> (o = g / Q, q = g % Q); element e at base + e*ES.
template <int DIR>
__global__ void k_lines(const double2* in, double2* out, Plan1D p, int n_in, int n_out,
                        long long ES_in, long long ES_out, int Q, long long nlines,
                        long long OS_in, long long OS_out, int NL, const int* __restrict__ halt) {
    if (halt && *halt) return;
    extern __shared__ double2 sm[];
    const int L = p.L, ld = L + 1;
    double2* a = sm;
    double2* b = sm + NL * ld;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const long long g0 = (long long)blockIdx.x * NL;
    for (int u = tid; u < NL * L; u += nthr) {
        const int l = u % NL, e = u / NL;
        const long long g = g0 + l;
        double2 v = make_double2(0.0, 0.0);
        if (g < nlines && e < n_in) {
            const long long o = g / Q, q = g - o * Q;
            v = in[o * OS_in + q + e * ES_in];
        }
        a[l * ld + e] = v;
    }
    __syncthreads();
    double2* r = fft_lines<DIR>(a, b, NL, p, tid, nthr);
    for (int u = tid; u < NL * n_out; u += nthr) {
        const int l = u % NL, e = u / NL;
        const long long g = g0 + l;
        if (g >= nlines) continue;
        const long long o = g / Q, q = g - o * Q;
        out[o * OS_out + q + e * ES_out] = r[l * ld + e];
    }
}

// P3: forward transform along the outer axis, 3x3 symmetric multiply with
// the kernel spectra (XX,XY,XZ,YY,YZ,ZZ; demag.py:33-34,211-215), inverse
// transform, keep n outputs.  In place in X.
__global__ void k_fused(double2* X, const double2* __restrict__ K, Plan1D p, int n,
                        long long ES, int hx, int hxp, int G, long long GS, int NK, double scale,
                        const int* __restrict__ halt) {
    if (halt && *halt) return;
    extern __shared__ double2 sm[];
    const int L = p.L, ld = L + 1;
    const int NL = 3 * NK;
    double2* a = sm;
    double2* b = sm + NL * ld;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int g = blockIdx.y;
    const int kx0 = blockIdx.x * NK;
    for (int u = tid; u < NL * L; u += nthr) {
        const int l = u % NL, e = u / NL;
        const int kx = kx0 + l / 3, c = l % 3;
        double2 v = make_double2(0.0, 0.0);
        if (kx < hx && e < n) v = X[g * GS + (long long)kx * 3 + c + e * ES];
        a[l * ld + e] = v;
    }
    __syncthreads();
    double2* r = fft_lines<-1>(a, b, NL, p, tid, nthr);
    double2* o = (r == a) ? b : a;
    for (int u = tid; u < NK * L; u += nthr) {
        const int kl = u % NK, e = u / NK;
        const int kx = kx0 + kl;
        if (kx >= hx) continue;
        const double2* k6 = K + (((long long)e * G + g) * hxp + kx) * 6;
        const double2 kxx = k6[0], kxy = k6[1], kxz = k6[2], kyy = k6[3], kyz = k6[4], kzz = k6[5];
        double2* s0 = r + (3 * kl) * ld + e;
        const double2 m0 = s0[0], m1 = s0[ld], m2 = s0[2 * ld];
        double2 h0 = cadd(cadd(cmul(kxx, m0), cmul(kxy, m1)), cmul(kxz, m2));
        double2 h1 = cadd(cadd(cmul(kxy, m0), cmul(kyy, m1)), cmul(kyz, m2));
        double2 h2 = cadd(cadd(cmul(kxz, m0), cmul(kyz, m1)), cmul(kzz, m2));
        s0[0] = make_double2(h0.x * scale, h0.y * scale);
        s0[ld] = make_double2(h1.x * scale, h1.y * scale);
        s0[2 * ld] = make_double2(h2.x * scale, h2.y * scale);
    }
    __syncthreads();
    double2* w = fft_lines<1>(r, o, NL, p, tid, nthr);
    for (int u = tid; u < NL * n; u += nthr) {
        const int l = u % NL, e = u / NL;
        const int kx = kx0 + l / 3, c = l % 3;
        if (kx < hx) X[g * GS + (long long)kx * 3 + c + e * ES] = w[l * ld + e];
    }
}

// P5: Hermitian-extend the hx bins to L, inverse FFT, keep n_out real values.
__global__ void k_rows_c2r(const double2* __restrict__ X, int hxp, int hx, int nc,
                           double* __restrict__ out, long long out_cstride, int out_pitch,
                           int n_out, int nrows, Plan1D p, int NL, const int* __restrict__ halt) {
    if (halt && *halt) return;
    extern __shared__ double2 sm[];
    const int L = p.L, ld = L + 1;
    double2* a = sm;
    double2* b = sm + NL * ld;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const long long line0 = (long long)blockIdx.x * NL;
    const int rows_here = NL / nc;
    const long long row0 = line0 / nc;
    for (int u = tid; u < rows_here * hx * nc; u += nthr) {
        const int rl = u / (hx * nc), q = u - rl * (hx * nc);
        const int kx = q / nc, c = q - kx * nc;
        const long long row = row0 + rl;
        double2 v = make_double2(0.0, 0.0);
        if (row < nrows) v = X[(row * hxp + kx) * nc + c];
        double2* s = a + (rl * nc + c) * ld;
        s[kx] = v;
        if (kx > 0 && L - kx >= hx) s[L - kx] = make_double2(v.x, -v.y);
    }
    __syncthreads();
    double2* r = fft_lines<1>(a, b, NL, p, tid, nthr);
    for (int u = tid; u < NL * n_out; u += nthr) {
        const int l = u / n_out, e = u - l * n_out;
        const long long gl = line0 + l;
        const long long row = gl / nc;
        const int c = (int)(gl - row * nc);
        if (row >= nrows) continue;
        out[c * out_cstride + row * out_pitch + e] = r[l * ld + e].x;
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

static const int kThreads = 256;
static const size_t kSmemBudget = 100 * 1024;
static const size_t kSmemMax = 200 * 1024;

static int lines_per_block(int L, int multiple, size_t budget = kSmemBudget) {
    size_t per = 2 * (size_t)(L + 1) * sizeof(double2);
    int nl = (int)std::max<size_t>(1, budget / per);
    nl = std::min(nl, 64);
    nl = std::max(multiple, (nl / multiple) * multiple);
    return nl;
}

static int set_smem_attrs() {
    static bool done = false;
    if (done) return MXB_OK;
    MXB_CUDA(cudaFuncSetAttribute(k_rows_r2c, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax));
    MXB_CUDA(cudaFuncSetAttribute(k_lines<-1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax));
    MXB_CUDA(cudaFuncSetAttribute(k_lines<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax));
    MXB_CUDA(cudaFuncSetAttribute(k_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax));
    MXB_CUDA(cudaFuncSetAttribute(k_rows_c2r, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax));
    done = true;
    return MXB_OK;
}

static size_t smem_for(int L, int NL) { return 2 * (size_t)NL * (L + 1) * sizeof(double2); }

int launch_rows_r2c(const Plan1D& p, const double* in, long long in_cstride, int in_pitch,
                    int n_in, double2* out, int hxp, int hx, int nc, long long nrows,
                    cudaStream_t st, const int* halt, int ostride, int coff) {
    if (ostride <= 0) ostride = nc;
    int NL = lines_per_block(p.L, nc);
    size_t sm = smem_for(p.L, NL);
    if (sm > kSmemMax) { set_error("x transform length too large for the generic path"); return MXB_EINVAL; }
    long long nlines = nrows * nc;
    unsigned nb = (unsigned)((nlines + NL - 1) / NL);
    k_rows_r2c<<<nb, kThreads, sm, st>>>(in, in_cstride, in_pitch, n_in, out, hxp, hx, nc,
                                         ostride, coff, (int)nrows, p, NL, halt);
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

int launch_lines(int dir, const Plan1D& p, const double2* in, double2* out, int n_in, int n_out,
                 long long ES_in, long long ES_out, int Q, long long nlines, long long OS_in,
                 long long OS_out, cudaStream_t st, const int* halt) {
    int NL = lines_per_block(p.L, 8);
    if (smem_for(p.L, NL) > kSmemMax) NL = lines_per_block(p.L, 1, kSmemMax);
    size_t sm = smem_for(p.L, NL);
    if (sm > kSmemMax) { set_error("line transform length too large for the generic path"); return MXB_EINVAL; }
    unsigned nb = (unsigned)((nlines + NL - 1) / NL);
    if (dir < 0)
        k_lines<-1><<<nb, kThreads, sm, st>>>(in, out, p, n_in, n_out, ES_in, ES_out, Q, nlines,
                                              OS_in, OS_out, NL, halt);
    else
        k_lines<1><<<nb, kThreads, sm, st>>>(in, out, p, n_in, n_out, ES_in, ES_out, Q, nlines,
                                             OS_in, OS_out, NL, halt);
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

int launch_fused(const Plan1D& p, double2* X, const double2* K, int n, long long ES, int hx,
                 int hxp, int G, long long GS, double scale, cudaStream_t st, const int* halt) {
    int NK = std::max(1, lines_per_block(p.L, 3) / 3);
    NK = std::min(NK, 8);
    size_t sm = smem_for(p.L, 3 * NK);
    if (sm > kSmemMax) { set_error("fused transform length too large for the generic path"); return MXB_EINVAL; }
    dim3 grid((hx + NK - 1) / NK, G);
    k_fused<<<grid, kThreads, sm, st>>>(X, K, p, n, ES, hx, hxp, G, GS, NK, scale, halt);
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

int launch_rows_c2r(const Plan1D& p, const double2* X, int hxp, int hx, int nc, double* out,
                    long long out_cstride, int out_pitch, int n_out, long long nrows,
                    cudaStream_t st, const int* halt) {
    int NL = lines_per_block(p.L, nc);
    size_t sm = smem_for(p.L, NL);
    if (sm > kSmemMax) { set_error("x transform length too large for the generic path"); return MXB_EINVAL; }
    long long nlines = nrows * nc;
    unsigned nb = (unsigned)((nlines + NL - 1) / NL);
    k_rows_c2r<<<nb, kThreads, sm, st>>>(X, hxp, hx, nc, out, out_cstride, out_pitch, n_out,
                                         (int)nrows, p, NL, halt);
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

int DemagPlan::init(const mxb_grid& gr, int device, int nranks, int rk) {
    dev = device;
    g.nx = (int)gr.nx; g.ny = (int)gr.ny; g.nz = (int)gr.nz;
    g.N = (long long)gr.nx * gr.ny * gr.nz;
    g.dx = gr.dx; g.dy = gr.dy; g.dz = gr.dz;
    px = g.nx > 1 ? 2 * g.nx : 1;
    py = g.ny > 1 ? 2 * g.ny : 1;
    pz = g.nz > 1 ? 2 * g.nz : 1;
    hx = px / 2 + 1;
    hxp = (hx + 7) / 8 * 8;
    scale = 1.0 / ((double)px * (double)py * (double)pz);
    if (nranks < 1 || rk < 0 || rk >= nranks || g.nz % nranks != 0) {
        set_error("slab decomposition needs nz divisible by the number of ranks");
        return MXB_EINVAL;
    }
    G = nranks;
    rank = rk;
    nz_l = g.nz / G;
    z0 = rank * nz_l;
    if (G == 1) {
        CH = hx;
        CHP = hxp;
    } else {
        CH = (hx + G - 1) / G;
        CHP = (CH + 7) / 8 * 8;
        if (px < 4 || (px & (px - 1)) || (g.nx % 2)) {
            set_error("the slab decomposition needs a power-of-two nx (fast x passes)");
            return MXB_EINVAL;
        }
    }
    kx0 = rank * CH;
    kxn = std::max(0, std::min(CH, hx - kx0));
    blk = (long long)nz_l * g.ny * CHP * 3;
    xblk = blk;
    MXB_CUDA(cudaSetDevice(dev));
    int rc = set_smem_attrs();
    if (rc) return rc;
    if ((rc = make_plan(px, dev, &plx, &tw[0]))) return rc;
    if ((rc = make_plan(py, dev, &ply, &tw[1]))) return rc;
    if ((rc = make_plan(pz, dev, &plz, &tw[2]))) return rc;
    if (px >= 4 && (rc = make_plan(px / 2, dev, &plm, &twm))) return rc;
    const size_t xs = (size_t)G * blk;
    const size_t x2 = (size_t)g.nz * py * CHP * 3;
    MXB_CUDA(cudaMalloc(&XS, xs * sizeof(double2)));
    if (G > 1) MXB_CUDA(cudaMalloc(&XR, xs * sizeof(double2)));
    else XR = XS;
    bytes = xs * (G > 1 ? 2 : 1) * sizeof(double2);
    // the y/z intermediate of the 5-pass layout; a plane-pipeline candidate
    // allocates it only if finish_spectra does not select the pipeline
    if (pz > 1 && py > 1) {
        if (!pipe_candidate()) {
            MXB_CUDA(cudaMalloc(&X2, x2 * sizeof(double2)));
            bytes += x2 * sizeof(double2);
        }
    } else {
        X2 = XR;
    }
    return MXB_OK;
}

// shapes the plane pipeline covers (single rank, 3-D, ny == nz, power-of-two
// padding, fast x rows); MXB_PIPE=0 disables it, MXB_PIPE=1 lifts the size floor
bool DemagPlan::pipe_candidate(bool symmetric) const {
    if (pz <= 1 || py <= 1 || !fast) return false;
    // z slab: the pipeline runs on the rank's kx chunk of all nz planes, read in
    // place from the all-to-all receive blocks (pairs of rows need even nz_l)
    if (G > 1 && (nz_l < 2 || (nz_l & (nz_l - 1)))) return false;
    if (px < 4 || (px & (px - 1)) || (g.nx % 2)) return false;
    if (!pipe_shape_ok(g.ny, g.nz)) return false;
    if (!symmetric && !pipe_cplx_ok(pz)) return false;
    const char* e = getenv("MXB_PIPE");
    if (e && e[0] == '0') return false;
    if (e && e[0] == '1') return true;
    // measured on B200 with the warp-FFT pipelines: 23.9 vs 34.4 ms for the y/z
    // part at 512^3 (L = 1024), 4.03 vs 4.55 ms at 256^3 (L = 512); slower below
    return pz >= 512;
}

// long y lines beyond the pipeline (py = 2048 / 4096, e.g. the 2048^2 x 64
// film): plane-major spectra, row kernels for y, the fused z pass over
// ky-contiguous chunks.  MXB_LONGY=0 keeps the 5-pass column kernels.
bool DemagPlan::longy_candidate() const {
    if (pz <= 1 || !fast || pipe) return false;
    if (G > 1 && (nz_l < 1 || (nz_l & (nz_l - 1)))) return false;
    if (px < 4 || (px & (px - 1)) || (g.nx % 2)) return false;
    if (!longy_shape_ok(py) || !fast_fused_ok(pz)) return false;
    const char* e = getenv("MXB_LONGY");
    return !(e && e[0] == '0');
}

void DemagPlan::release() {
    cudaSetDevice(dev);
    for (auto& t : tw) if (t) cudaFree(t);
    if (twm) cudaFree(twm);
    if (Kq) cudaFree(Kq);
    if (Kp) cudaFree(Kp);
    if (slots) cudaFree(slots);
    if (bar) cudaFree(bar);
    Kp = nullptr;
    slots = nullptr;
    bar = nullptr;
    if (Kc && Kc != K) cudaFree(Kc);
    if (K) cudaFree(K);
    if (T) cudaFree(T);
    T = nullptr;
    if (X2 && X2 != XR) cudaFree(X2);
    if (XR && XR != XS) cudaFree(XR);
    if (XS) cudaFree(XS);
    XS = XR = X2 = K = Kc = nullptr;
    Kq = nullptr;
    twm = nullptr;
}

// The spectra are built per rank: one rank keeps all hx planes; a slab rank
// (G > 1) transforms each component along x into a one-component scratch T and
// keeps only its kx chunk, so the y/z transforms and the build memory scale
// with hx/G (the 2048^2 x 64 film: ~17 + 13 GB per rank instead of 103 GB).
static int alloc_full_spectra(DemagPlan& p, cudaStream_t st) {
    if (p.K) return MXB_OK;
    p.kpitch = p.G > 1 ? p.CHP : p.hxp;
    p.koff = p.G > 1 ? p.kx0 : 0;
    const size_t n = (size_t)p.pz * p.py * p.kpitch * 6;
    MXB_CUDA(cudaMalloc(&p.K, n * sizeof(double2)));
    MXB_CUDA(cudaMemsetAsync(p.K, 0, n * sizeof(double2), st));
    if (p.G > 1 && !p.T) MXB_CUDA(cudaMalloc(&p.T, (size_t)p.pz * p.py * p.hxp * sizeof(double2)));
    return MXB_OK;
}

// one component's kx chunk [kx0, kx0 + kxn) of the full x spectrum into slot c of K
__global__ void k_take_chunk(const double2* __restrict__ T, double2* __restrict__ K, long long nzy, int hxp,
                             int kx0, int kxn, int kpitch, int c) {
    const long long tot = nzy * kpitch;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot;
         t += (long long)gridDim.x * blockDim.x) {
        const int kx = (int)(t % kpitch);
        const long long zy = t / kpitch;
        K[t * 6 + c] = kx < kxn ? T[zy * hxp + kx0 + kx] : make_double2(0.0, 0.0);
    }
}

// x r2c of one packed real-space component (pz,py,px) into slot c of K
int DemagPlan::spectra_x_component(const double* Pc, int c, cudaStream_t st) {
    int rc = alloc_full_spectra(*this, st);
    if (rc) return rc;
    const long long plane = (long long)pz * py;
    if (G == 1) return launch_rows_r2c(plx, Pc, 0, px, px, K, hxp, hx, 1, plane, st, nullptr, 6, c);
    if ((rc = launch_rows_r2c(plx, Pc, 0, px, px, T, hxp, hx, 1, plane, st, nullptr, 1, 0))) return rc;
    k_take_chunk<<<148 * 8, 256, 0, st>>>(T, K, plane, hxp, kx0, kxn, kpitch, c);
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

// y and z forward transforms of all 6 slots of K, in place
int DemagPlan::spectra_yz(cudaStream_t st) {
    int rc;
    const int kp = kpitch;
    if (py > 1) {
        // y lines: element stride kp*6, Q = kp*6 per z-plane
        rc = launch_lines(-1, ply, K, K, py, py, (long long)kp * 6, (long long)kp * 6, kp * 6,
                          (long long)pz * kp * 6, (long long)py * kp * 6, (long long)py * kp * 6,
                          st, nullptr);
        if (rc) return rc;
    }
    if (T) { cudaFree(T); T = nullptr; }
    if (pz > 1) {
        long long Q = (long long)py * kp * 6;
        rc = launch_lines(-1, plz, K, K, pz, pz, Q, Q, (int)Q, Q, 0, 0, st, nullptr);
        if (rc) return rc;
    }
    return MXB_OK;
}

// 6 forward transforms of a packed (6,pz,py,px) device tensor into K.
int DemagPlan::spectra_from_packed_dev(const double* P, cudaStream_t st) {
    const long long per = (long long)pz * py * px;
    for (int c = 0; c < 6; ++c) {
        int rc = spectra_x_component(P + c * per, c, st);
        if (rc) return rc;
    }
    return spectra_yz(st);
}

// the rank's kx chunk of the complex spectra
__global__ void k_chunk_complex(const double2* K, double2* Kc, long long nzy, int hxp, int kx0,
                                int kxn, int CHP) {
    const long long tot = nzy * CHP * 6;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot;
         t += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(t % 6);
        long long r = t / 6;
        const int kx = (int)(r % CHP);
        const long long zy = r / CHP;
        Kc[t] = kx < kxn ? K[(zy * hxp + kx0 + kx) * 6 + c] : make_double2(0.0, 0.0);
    }
}

// real parts of the (exactly real, parity-structured) spectra, quarter storage
__global__ void k_quarterize(const double2* K, double* Kq, int L, int G, int py, int hxp,
                             int e_is_z, int kx0, int kxn, int CHP) {
    const int L2 = L / 2 + 1, G2 = G / 2 + 1;
    const long long tot = (long long)L2 * G2 * CHP * 6;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot;
         t += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(t % 6);
        long long r = t / 6;
        const int kx = (int)(r % CHP);
        r /= CHP;
        const int g2 = (int)(r % G2), e2 = (int)(r / G2);
        const int kz = e_is_z ? e2 : g2, ky = e_is_z ? g2 : e2;
        Kq[t] = kx < kxn ? K[(((long long)kz * py + ky) * hxp + kx0 + kx) * 6 + c].x : 0.0;
    }
}

int DemagPlan::finish_spectra(bool symmetric, cudaStream_t st) {
    const int L = fused_L(), GG = fused_G();
    if (Kq) { cudaFree(Kq); Kq = nullptr; }
    if (Kc && Kc != K) { cudaFree(Kc); }
    Kc = nullptr;
    kmode = 0;
    pipe = false;
    longy = false;
    if (Kp) { cudaFree(Kp); Kp = nullptr; }
    if (slots) { cudaFree(slots); slots = nullptr; }
    if (bar) { cudaFree(bar); bar = nullptr; }
    if (G == 1) {   // standard row layout unless the pipeline is selected below
        CH = hx;
        CHP = hxp;
        blk = (long long)nz_l * g.ny * CHP * 3;
    }
    xblk = blk;
    if (pipe_candidate(symmetric)) {
        // plane-major spectra, slot ring, barrier; x passes switch to [kx][z][y][3].
        // Symmetric (mirrored) tensor: real parity-reduced quarter Kp[kx][ky'][kz'][6];
        // otherwise (the reference's tensor via from_packed, or the unmirrored GPU
        // build) the full complex rows Kp[kx][ky][kz][6] (8x the bytes, no symmetry assumed)
        // Slab (G ranks): planes [kx0, kx0 + kxn) of CHr per rank; the x passes write
        // plane-major [kx][z_l][y][3] (CHr planes per all-to-all block, so each block
        // is contiguous), and the pipeline reads the received [g][kx][z_l][y][3].
        const int L2 = pz / 2 + 1;
        const int CHr = G == 1 ? hx : (hx + G - 1) / G;
        kx0 = rank * CHr;
        kxn = std::max(0, std::min(CHr, hx - kx0));
        const size_t np = (size_t)std::max(kxn, 1);
        const size_t nk = symmetric ? np * L2 * L2 * 6 : np * pz * pz * 12;
        const size_t ns = (size_t)3 * g.nz * py * 3;
        MXB_CUDA(cudaMalloc(&Kp, nk * sizeof(double)));
        MXB_CUDA(cudaMalloc(&slots, ns * sizeof(double2)));
        MXB_CUDA(cudaMalloc(&bar, (2 + 3 * (size_t)hx + 3 * (size_t)g.nz) * sizeof(unsigned)));
        int rc = MXB_OK;
        if (kxn > 0)
            rc = symmetric ? pipe_quarter(K, Kp, pz, kxn, kpitch, st, kx0 - koff)
                           : pipe_complex(K, reinterpret_cast<double2*>(Kp), pz, kxn, kpitch, st, kx0 - koff);
        if (rc) return rc;
        CH = 1;
        CHP = 1;
        blk = (long long)CHr * nz_l * g.ny * 3;
        xblk = (long long)nz_l * g.ny * 3;
        kmode = symmetric ? 3 : 5;
        pipe = true;
        MXB_CUDA(cudaStreamSynchronize(st));
        cudaFree(K);
        K = nullptr;
        bytes += nk * sizeof(double) + ns * sizeof(double2);
        has_kernel = true;
        return MXB_OK;
    }
    if (symmetric && longy_candidate()) {
        // plane-major XR [kx][z][y][3] and X2 [kx][z][ky][3] (both fit the
        // row-major allocations), kernel Kp[kx][ky'][kz'][6]
        // (on a z slab: the rank's kx chunk of CHr planes, XR the all-to-all receive blocks)
        const int CHr = G == 1 ? hx : (hx + G - 1) / G;
        kx0 = rank * CHr;
        kxn = std::max(0, std::min(CHr, hx - kx0));
        const size_t nk = (size_t)std::max(kxn, 1) * (py / 2 + 1) * (pz / 2 + 1) * 6;
        MXB_CUDA(cudaMalloc(&Kp, nk * sizeof(double)));
        int rc = kxn > 0 ? longy_quarter(K, Kp, py, pz, kxn, kpitch, st, kx0 - koff) : MXB_OK;
        if (rc) return rc;
        if (!X2) {
            const size_t x2 = (size_t)g.nz * py * CHP * 3;
            MXB_CUDA(cudaMalloc(&X2, x2 * sizeof(double2)));
            bytes += x2 * sizeof(double2);
        }
        CH = 1;
        CHP = 1;
        blk = (long long)CHr * nz_l * g.ny * 3;
        xblk = (long long)nz_l * g.ny * 3;
        kmode = 4;
        longy = true;
        MXB_CUDA(cudaStreamSynchronize(st));
        cudaFree(K);
        K = nullptr;
        bytes += nk * sizeof(double);
        has_kernel = true;
        return MXB_OK;
    }
    if (pz > 1 && py > 1 && !X2) {
        const size_t x2 = (size_t)g.nz * py * CHP * 3;
        MXB_CUDA(cudaMalloc(&X2, x2 * sizeof(double2)));
        bytes += x2 * sizeof(double2);
    }
    if (symmetric && fast_fused_ok(L)) {
        const int e_is_z = pz > 1 ? 1 : (py > 1 ? 0 : 1);
        const size_t n = (size_t)(L / 2 + 1) * (GG / 2 + 1) * CHP * 6;
        MXB_CUDA(cudaMalloc(&Kq, n * sizeof(double)));
        k_quarterize<<<148 * 8, 256, 0, st>>>(K, Kq, L, GG, py, kpitch, e_is_z, kx0 - koff, kxn, CHP);
        MXB_LAUNCH_CHECK();
        kmode = 2;
    } else if (G == 1 || (kpitch == CHP && koff == kx0)) {
        Kc = K;   // the chunk is the whole (rank-built) spectrum
    } else {
        const size_t n = (size_t)pz * py * CHP * 6;
        MXB_CUDA(cudaMalloc(&Kc, n * sizeof(double2)));
        k_chunk_complex<<<148 * 8, 256, 0, st>>>(K, Kc, (long long)pz * py, kpitch, kx0 - koff, kxn, CHP);
        MXB_LAUNCH_CHECK();
    }
    MXB_CUDA(cudaStreamSynchronize(st));
    if (Kc != K) {
        cudaFree(K);
        K = nullptr;
    }
    bytes += kmode == 2 ? (size_t)(L / 2 + 1) * (GG / 2 + 1) * CHP * 6 * sizeof(double)
                        : (size_t)pz * py * CHP * 6 * sizeof(double2);
    has_kernel = true;
    return MXB_OK;
}

int DemagPlan::x_forward(const double* m, cudaStream_t st, const int* halt) {
    const long long Nl = (long long)nz_l * g.ny * g.nx;
    const long long rows = (long long)nz_l * g.ny;
    const int nx = g.nx;
    int rc = -1;
    static const bool rm_t = !(getenv("MXB_LONGY_RMT") && getenv("MXB_LONGY_RMT")[0] == '0');
    if (longy && rm_t && G == 1) {
        // row-major r2c into X2 (free until the y forward), then a tiled transpose
        // into the plane-major XR (longy.cu)
        rc = fast_rows(true, px / 2, m, X2, nullptr, Nl, nx, nx / 2, hx, hxp, (long long)g.nz * g.ny * hxp * 3, rows,
                       plm.tw, plx.tw, st, halt);
        if (rc == -1) { set_error("no x kernel for the long-y path"); return MXB_EINVAL; }
        if (rc) return rc;
        return longy_rm_to_pm(X2, XS, g.ny, g.nz, hx, hxp, st);
    }
    if (fast && px >= 4 && (nx % 2) == 0)
        rc = fast_rows(true, px / 2, m, XS, nullptr, Nl, nx, nx / 2, CH, CHP, xblk, rows, plm.tw,
                       plx.tw, st, halt);
    if (rc == -1) {
        if (G > 1) { set_error("no x kernel for this slab shape"); return MXB_EINVAL; }
        rc = launch_rows_r2c(plx, m, Nl, nx, nx, XS, hxp, hx, 3, rows, st, halt, 3, 0);
    }
    return rc;
}

int DemagPlan::x_inverse(double* h, cudaStream_t st, const int* halt) {
    const long long Nl = (long long)nz_l * g.ny * g.nx;
    const long long rows = (long long)nz_l * g.ny;
    const int nx = g.nx;
    int rc = -1;
    if (fast && px >= 4 && (nx % 2) == 0)
        rc = fast_rows(false, px / 2, nullptr, XS, h, Nl, nx, nx / 2, CH, CHP, xblk, rows, plm.tw,
                       plx.tw, st, halt);
    if (rc == -1) {
        if (G > 1) { set_error("no x kernel for this slab shape"); return MXB_EINVAL; }
        rc = launch_rows_c2r(plx, XS, hxp, hx, 3, h, Nl, nx, nx, rows, st, halt);
    }
    return rc;
}

// y forward, fused z (or y) multiply, y inverse on the kx chunk held in XR
int DemagPlan::yz(cudaStream_t st, const int* halt, cudaEvent_t* ev) {
    auto mark = [&](int i) { if (ev) cudaEventRecord(ev[i], st); };
    if (!has_kernel) { set_error("demag kernel has no spectra (call set_packed or build)"); return MXB_EINVAL; }
    const int ny = g.ny, nz = g.nz;
    const long long row = (long long)CHP * 3;   // complex elements per (z,y) row of the chunk
    int rc;
    if (kxn <= 0) { mark(2); mark(3); mark(4); return MXB_OK; }
    if (pipe) {
        mark(2);
        rc = pipe_yz(XR, slots, Kp, bar, kxn, nz, scale, plz.tw, st, halt, kmode == 5 ? 1 : 0, nz_l, blk);
        mark(3);
        mark(4);
        return rc;
    }
    if (longy) {
        // y forward (rows (kx, z): ny -> py), fused z over ky-contiguous tiles, y inverse
        const long long rows = (long long)kxn * nz;   // the rank's planes (all hx on one rank)
        if ((rc = longy_rows(-1, py, XR, X2, ny, py, rows, ply.tw, st, halt, nz, nz_l, blk))) return rc;
        mark(2);
        FusedArgs a{X2, Kp, nz, (long long)py * 3, py, 0, kxn, (long long)nz * py * 3, scale, 1};
        rc = fast_fused(pz, 4, a, plz.tw, st, halt);
        if (rc == -1) { set_error("no fused kernel for this shape"); rc = MXB_EINVAL; }
        if (rc) return rc;
        mark(3);
        if ((rc = longy_rows(1, py, X2, XR, py, ny, rows, ply.tw, st, halt, nz, nz_l, blk))) return rc;
        mark(4);
        return MXB_OK;
    }
    auto cols = [&](int dir, const double2* in, double2* out, int n_in, int n_out, long long OS_in,
                    long long OS_out) {
        int r = -1;
        if (fast) r = fast_cols(dir, py, in, out, n_in, n_out, row, row, kxn * 3, (long long)nz * kxn * 3,
                                OS_in, OS_out, ply.tw, st, halt);
        if (r == -1) r = launch_lines(dir, ply, in, out, n_in, n_out, row, row, kxn * 3,
                                      (long long)nz * kxn * 3, OS_in, OS_out, st, halt);
        return r;
    };
    auto fused = [&](const Plan1D& pl, double2* X, int n, long long ES, int GG, long long GS, int e_is_z) {
        int r = -1;
        if (fast || kmode != 0) {
            FusedArgs a{X, kmode == 0 ? (const void*)Kc : (const void*)Kq, n, ES, kxn, CHP, GG, GS, scale, e_is_z};
            r = fast_fused(pl.L, kmode, a, pl.tw, st, halt);
        }
        if (r == -1 && kmode == 0) r = launch_fused(pl, X, Kc, n, ES, kxn, CHP, GG, GS, scale, st, halt);
        if (r == -1) { set_error("no fused kernel for this shape"); r = MXB_EINVAL; }
        return r;
    };
    if (pz > 1) {
        if (py > 1 && (rc = cols(-1, XR, X2, ny, py, (long long)ny * row, (long long)py * row))) return rc;
        mark(2);
        if ((rc = fused(plz, X2, nz, (long long)py * row, py, row, 1))) return rc;
        mark(3);
        if (py > 1 && (rc = cols(1, X2, XR, py, ny, (long long)py * row, (long long)ny * row))) return rc;
        mark(4);
    } else if (py > 1) {
        mark(2);
        if ((rc = fused(ply, XR, ny, row, 1, 0, 0))) return rc;
        mark(3);
        mark(4);
    } else {
        mark(2);
        if ((rc = fused(plz, XR, 1, row, 1, 0, 1))) return rc;
        mark(3);
        mark(4);
    }
    return MXB_OK;
}

int DemagPlan::check_abort() {
    if (!pipe || !bar) return MXB_OK;
    unsigned w = 0;
    MXB_CUDA(cudaMemcpy(&w, bar + 1, sizeof(unsigned), cudaMemcpyDeviceToHost));
    if (w) {
        set_error("demag plane pipeline: dependency wait timed out (scheduling fault); field invalid");
        return MXB_ECUDA;
    }
    return MXB_OK;
}

int DemagPlan::field_dev(const double* m, double* h, cudaStream_t st, const int* halt,
                         cudaEvent_t* ev) {
    if (G != 1) { set_error("field_dev is the single-rank pipeline"); return MXB_EINVAL; }
    if (!has_kernel) { set_error("demag kernel has no spectra (call set_packed or build)"); return MXB_EINVAL; }
    // MXB_SYNC_DEBUG=1: synchronise after every pass and name the one that failed
    static const bool dbg = getenv("MXB_SYNC_DEBUG") != nullptr;
    auto sync = [&](const char* what) -> int {
        if (!dbg) return MXB_OK;
        cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return cuda_fail(e, what, __FILE__, __LINE__);
        return MXB_OK;
    };
    if (ev) cudaEventRecord(ev[0], st);
    int rc = x_forward(m, st, halt);
    if (rc || (rc = sync("x_forward"))) return rc;
    if (ev) cudaEventRecord(ev[1], st);
    if ((rc = yz(st, halt, ev)) || (rc = sync("yz"))) return rc;
    rc = x_inverse(h, st, halt);
    if (!rc) rc = sync("x_inverse");
    if (ev) cudaEventRecord(ev[5], st);
    return rc;
}

}  // namespace mxb
