// Internal definitions shared by the libmagnex_b200 translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/magnex_b200.h"

#define MXB_MU0 (4.0e-7 * 3.141592653589793)

namespace mxb {

void set_error(const std::string& msg);
int cuda_fail(cudaError_t e, const char* what, const char* file, int line);

#define MXB_CUDA(call)                                                    \
    do {                                                                  \
        cudaError_t e_ = (call);                                          \
        if (e_ != cudaSuccess) return mxb::cuda_fail(e_, #call, __FILE__, __LINE__); \
    } while (0)

#define MXB_LAUNCH_CHECK()                                                \
    do {                                                                  \
        cudaError_t e_ = cudaGetLastError();                              \
        if (e_ != cudaSuccess) return mxb::cuda_fail(e_, "kernel launch", __FILE__, __LINE__); \
    } while (0)

// --- arithmetic with optional "reference order" semantics --------------------
// In exact mode every op is an explicitly rounded intrinsic, so nvcc cannot
// contract a*b+c into an FMA; results then follow numpy's per-op rounding.
template <bool E> __device__ __forceinline__ double add(double a, double b) {
    return E ? __dadd_rn(a, b) : a + b;
}
template <bool E> __device__ __forceinline__ double sub(double a, double b) {
    return E ? __dsub_rn(a, b) : a - b;
}
template <bool E> __device__ __forceinline__ double mul(double a, double b) {
    return E ? __dmul_rn(a, b) : a * b;
}
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }

struct Grid {
    int nx, ny, nz;
    long long N;
    double dx, dy, dz;
};

// Material as seen by kernels: scalars plus optional per-cell arrays.
struct MatDev {
    double Ms, A, Ku, D, alpha, gamma;
    double ek[3];
    const double* Ms_c;
    const double* A_c;
    const double* Ku_c;
    const double* D_c;
    const double* alpha_c;
    const double* ek_c;
    double Kc1, c1[3], c2[3], c3[3], Db;
    int uniform;       // 1 if no per-cell array is set
    int all_magnetic;  // Ms > 0 everywhere
};

// Device-side control block for the fused stepping loop (reductions + stop flags).
struct Ctl {
    unsigned int arrive;   // last-block-done counter
    int halt;              // 0 run, MXB_EQUILIBRATED, MXB_EBLOWUP, MXB_EDEAD
    long long dead_flat;   // min flat index of a dead cell (LLONG_MAX if none)
    long long steps_done;  // committed steps in this run call
    double mean[3];        // <m> of the last committed step
    double prev_mean[3];
    double residual;
    double drift;
    double eq_tol;
    long long n_magnetic;
    double energies[4];
};

constexpr int kReduceSlots = 8;  // doubles per block partial

}  // namespace mxb
