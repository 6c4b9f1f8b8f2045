// Microbenchmark: throughput of the warp FFT building blocks on one B200,
// no global traffic in the loop (data stays in registers / shared memory).
#include <cstdio>
#include "../../paper_2602_12242_b200/csrc/fft_warp.cuh"
#include "../../paper_2602_12242_b200/csrc/fft_fast.cuh"
using namespace mxb;

template <int MODE>
__global__ void __launch_bounds__(96) kbench(double2* out, const double2* __restrict__ tw, int iters) {
    __shared__ double2 W[3 * 1024];
    const int c = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double2 v[32];
#pragma unroll
    for (int m = 0; m < 32; ++m) v[m] = make_double2(lane * 0.001 + m, c - m * 0.5);
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) fw::dft32<-1>(v);
        else fw::fft1024<-1>(v, W + c * 1024, lane, tw);
    }
    double2 s = make_double2(0, 0);
#pragma unroll
    for (int m = 0; m < 32; ++m) s = cadd(s, v[m]);
    out[blockIdx.x * 96 + threadIdx.x] = s;
}

// CTA-wide radix-16 core for comparison: 3 lines of 1024, 192 threads
__global__ void __launch_bounds__(192) kbench16(double2* out, const double2* __restrict__ tw, int iters) {
    extern __shared__ double2 X[];
    const int b = threadIdx.x / 64, t = threadIdx.x % 64;
    double2 v[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = make_double2(t * 0.001 + m, b - m * 0.5);
    for (int it = 0; it < iters; ++it) ff::fft_core<1024, 16, 3, false, -1>(v, X, b, t, tw);
    double2 s = make_double2(0, 0);
#pragma unroll
    for (int m = 0; m < 16; ++m) s = cadd(s, v[m]);
    out[blockIdx.x * 192 + threadIdx.x] = s;
}

int main() {
    double2 *out, *tw;
    cudaMalloc(&out, 148 * 64 * 192 * sizeof(double2));
    cudaMalloc(&tw, 1024 * sizeof(double2));
    double2 h[1024];
    for (int n = 0; n < 1024; ++n) h[n] = make_double2(cos(-2 * M_PI * n / 1024), sin(-2 * M_PI * n / 1024));
    cudaMemcpy(tw, h, sizeof h, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 200;
    for (int mode = 0; mode < 3; ++mode) {
        for (int ctas_per_sm : {1, 2, 3, 4}) {
            const int grid = 148 * ctas_per_sm;
            size_t sm16 = (size_t)ff::smem_elems<1024, 16, 3>() * sizeof(double2);
            if (mode == 2) cudaFuncSetAttribute(kbench16, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm16);
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                if (mode == 0) kbench<0><<<grid, 96>>>(out, tw, iters);
                else if (mode == 1) kbench<1><<<grid, 96>>>(out, tw, iters);
                else kbench16<<<grid, 192, sm16>>>(out, tw, iters);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
            }
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            cudaError_t err = cudaGetLastError();
            // work: lines of 1024 points (mode 0: 32-point DFTs per thread)
            double lines = (double)grid * 3 * iters;
            double pts = mode == 0 ? (double)grid * 96 * 32 * iters : lines * 1024;
            printf("%s ctas/sm=%d: %.3f ms  %.2f Gpoint/s  %.3f clk/point/SM  %s\n",
                   mode == 0 ? "dft32   " : (mode == 1 ? "warp1024" : "radix16 "), ctas_per_sm, ms,
                   pts / ms / 1e6, (ms * 1e-3 * 1.965e9 * 148) / pts, cudaGetErrorString(err));
        }
    }
    return 0;
}
