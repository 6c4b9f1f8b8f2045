// Measured FP64 FMA peak of this GPU (the denominator for the FP64-pipe
// figures in bench.py; SURVEY 8d asks for it because MEASURED_PEAKS has no
// FP64 entry).  8 independent DFMA chains per thread, 1024 iterations, grid
// = 8 CTAs of 256 threads per SM; best of 5 timed launches (CUDA events).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
//   ./fp64_peak  -> {"fp64_tflops": ..., "sm_count": ..., "clock_mhz": ...}
#include <cstdio>

constexpr int CH = 8, IT = 1024;

__global__ void __launch_bounds__(256) k_fma(double* out, double a, double b) {
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-9 + c;
    for (int i = 0; i < IT; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    if (s == 12345.678) out[0] = s;   // never true; keeps the chains live
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double* out;
    cudaMalloc(&out, 8);
    const int grid = sms * 8, block = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_fma<<<grid, block>>>(out, 0.999999, 1e-7);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        for (int k = 0; k < 20; ++k) k_fma<<<grid, block>>>(out, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double flops = 20.0 * grid * block * (double)CH * IT * 2.0;
    printf("{\"fp64_tflops\": %.2f, \"sm_count\": %d, \"clock_mhz_nominal\": %d, \"how\": \"%d CTAs x %d threads x %d "
           "chains x %d DFMA, 20 launches, best of 5, CUDA events\"}\n",
           flops / (best * 1e-3) / 1e12, sms, clk / 1000, grid, block, CH, IT);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
