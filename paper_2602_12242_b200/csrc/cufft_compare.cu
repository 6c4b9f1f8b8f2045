// cuFFT version of one demag evaluation -- a TIMED COMPARISON ONLY.
// It is never called on the product path; bench.py reports its time beside
// the hand-written pipeline (demag.cu) for the same grid and kernel.
#include <cufft.h>

#include "demag.cuh"

namespace mxb {

__global__ void k_pad3(const double* m, double* pad, int nx, int ny, int nz, int px, int py, int pz) {
    const long long tot = 3LL * px * py * pz;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot;
         t += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(t % px);
        long long r = t / px;
        const int y = (int)(r % py);
        r /= py;
        const int z = (int)(r % pz), c = (int)(r / pz);
        double v = 0.0;
        if (x < nx && y < ny && z < nz) v = m[(((long long)c * nz + z) * ny + y) * nx + x];
        pad[t] = v;
    }
}

__global__ void k_crop3(const double* pad, double* h, int nx, int ny, int nz, int px, int py, int pz,
                        double scale) {
    const long long tot = 3LL * nx * ny * nz;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot;
         t += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(t % nx);
        long long r = t / nx;
        const int y = (int)(r % ny);
        r /= ny;
        const int z = (int)(r % nz), c = (int)(r / nz);
        h[t] = pad[(((long long)c * pz + z) * py + y) * px + x] * scale;
    }
}

// the kernel spectra are exactly real (the Newell tensor is even, or odd in two
// axes): kept as six real planes, multiplied as real scalars
__global__ void k_kernel_soa(const double2* K, double* Ks, int pz, int py, int hx, int hxp) {
    const long long n = (long long)pz * py * hx;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < 6 * n;
         t += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(t / n);
        const long long p = t % n;
        const int kx = (int)(p % hx);
        const long long zy = p / hx;
        Ks[t] = K[(zy * hxp + kx) * 6 + c].x;
    }
}

__global__ void k_mul3(double2* M, const double* Ks, long long n) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
         t += (long long)gridDim.x * blockDim.x) {
        const double2 m0 = M[t], m1 = M[n + t], m2 = M[2 * n + t];
        double k[6];
        for (int c = 0; c < 6; ++c) k[c] = Ks[c * n + t];
        M[t] = make_double2(k[0] * m0.x + k[1] * m1.x + k[2] * m2.x, k[0] * m0.y + k[1] * m1.y + k[2] * m2.y);
        M[n + t] = make_double2(k[1] * m0.x + k[3] * m1.x + k[4] * m2.x, k[1] * m0.y + k[3] * m1.y + k[4] * m2.y);
        M[2 * n + t] = make_double2(k[2] * m0.x + k[4] * m1.x + k[5] * m2.x, k[2] * m0.y + k[4] * m1.y + k[5] * m2.y);
    }
}

}  // namespace mxb

using namespace mxb;

struct mxb_demag;
extern "C" int mxb_demag_field_dev(mxb_demag* d, const double* m, double* h);

// defined in api.cu
namespace mxb { DemagPlan* demag_plan_of(mxb_demag* d); cudaStream_t demag_stream_of(mxb_demag* d); }

extern "C" int mxb_time_demag_cufft(mxb_demag* d, int iters, double* ms_eval) {
    if (!d || iters < 1) { set_error("bad argument"); return MXB_EINVAL; }
    DemagPlan& p = *demag_plan_of(d);
    cudaStream_t st = demag_stream_of(d);
    if (!p.has_kernel || !p.XS) { set_error("no spectra (or a surrogate handle)"); return MXB_EINVAL; }
    cudaSetDevice(p.dev);
    const Grid& g = p.g;
    const long long real_n = (long long)p.px * p.py * p.pz;
    const long long spec_n = (long long)p.pz * p.py * p.hx;
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    const size_t need = (3 * g.N * 2 + 3 * real_n + 6 * spec_n) * sizeof(double) + 3 * spec_n * sizeof(double2);
    if (need * 3 / 2 > fr) { set_error("not enough free memory for the cuFFT comparison"); return MXB_EINVAL; }
    double *m = nullptr, *h = nullptr, *pad = nullptr;
    double2* spec = nullptr;
    double* Ks = nullptr;
    MXB_CUDA(cudaMalloc(&m, 3 * g.N * sizeof(double)));
    MXB_CUDA(cudaMalloc(&h, 3 * g.N * sizeof(double)));
    MXB_CUDA(cudaMalloc(&pad, 3 * real_n * sizeof(double)));
    MXB_CUDA(cudaMalloc(&spec, 3 * spec_n * sizeof(double2)));
    MXB_CUDA(cudaMalloc(&Ks, 6 * spec_n * sizeof(double)));
    cudaMemsetAsync(m, 0, 3 * g.N * sizeof(double), st);
    if (p.kmode == 0) {
        k_kernel_soa<<<148 * 8, 256, 0, st>>>(p.Kc, Ks, p.pz, p.py, p.hx, p.CHP);
    } else {
        // same data volume for timing; values unfolded from the quarter on the host side are
        // not needed for a timing comparison
        cudaMemsetAsync(Ks, 0, 6 * spec_n * sizeof(double), st);
    }
    cufftHandle fwd, inv;
    int dims[3] = {p.pz, p.py, p.px};
    int rank = 3;
    if (cufftPlanMany(&fwd, rank, dims, nullptr, 1, (int)real_n, nullptr, 1, (int)spec_n, CUFFT_D2Z, 3) != CUFFT_SUCCESS ||
        cufftPlanMany(&inv, rank, dims, nullptr, 1, (int)spec_n, nullptr, 1, (int)real_n, CUFFT_Z2D, 3) != CUFFT_SUCCESS) {
        set_error("cufft plan failed");
        return MXB_ECUDA;
    }
    cufftSetStream(fwd, st);
    cufftSetStream(inv, st);
    auto once = [&]() {
        k_pad3<<<148 * 8, 256, 0, st>>>(m, pad, g.nx, g.ny, g.nz, p.px, p.py, p.pz);
        cufftExecD2Z(fwd, pad, (cufftDoubleComplex*)spec);
        k_mul3<<<148 * 8, 256, 0, st>>>(spec, Ks, spec_n);
        cufftExecZ2D(inv, (cufftDoubleComplex*)spec, pad);
        k_crop3<<<148 * 8, 256, 0, st>>>(pad, h, g.nx, g.ny, g.nz, p.px, p.py, p.pz, p.scale);
    };
    for (int w = 0; w < 2; ++w) once();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    for (int i = 0; i < iters; ++i) once();
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    *ms_eval = ms / iters;
    cufftDestroy(fwd);
    cufftDestroy(inv);
    cudaFree(m); cudaFree(h); cudaFree(pad); cudaFree(spec); cudaFree(Ks);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    MXB_CUDA(cudaGetLastError());
    return MXB_OK;
}
