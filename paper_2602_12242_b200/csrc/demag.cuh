#pragma once

#include "common.cuh"
#include "fft_generic.cuh"

namespace mxb {

struct FusedArgs {
    double2* X;
    const void* K;
    int n;
    long long ES;
    int hx, hxp, G;
    long long GS;
    double scale;
    int e_is_z;   // the transformed axis: 1 -> z (3-D), 0 -> y (film)
};

int fast_cols(int dir, int L, const double2* in, double2* out, int n_in, int n_out,
              long long ES_in, long long ES_out, int Q, long long nlines, long long OS_in,
              long long OS_out, const double2* tw, cudaStream_t st, const int* halt);
bool fast_fused_ok(int L);
int fast_fused(int L, int kmode, const FusedArgs& a, const double2* tw, cudaStream_t st,
               const int* halt);
int fast_rows(bool fwd, int M, const double* in_r, double2* X, double* out_r, long long cstride,
              int pitch, int nhalf, int hxp, long long nrows, const double2* twM,
              const double2* tw2M, cudaStream_t st, const int* halt);

struct DemagPlan {
    int dev = 0;
    Grid g{};
    int px = 1, py = 1, pz = 1, hx = 1, hxp = 8;
    double scale = 1.0;
    Plan1D plx{}, ply{}, plz{};
    double2* tw[3] = {nullptr, nullptr, nullptr};
    double2* X1 = nullptr;   // [nz][ny][hxp][3]
    double2* X2 = nullptr;   // [nz][py][hxp][3]
    double2* K = nullptr;    // [pz][py][hxp][6] spectra (unscaled), complex
    double* Kq = nullptr;    // parity-reduced real spectra [L/2+1][G/2+1][hxp][6]
    int kmode = 0;           // 0 complex K, 2 real quarter Kq
    Plan1D plm{};            // length px/2 (fast x rows)
    double2* twm = nullptr;
    bool fast = true;        // use the register-resident kernels where shapes allow
    bool has_kernel = false;
    int fused_L() const { return pz > 1 ? pz : (py > 1 ? py : 1); }
    int fused_G() const { return pz > 1 ? py : 1; }
    int quarterize(cudaStream_t st);
    size_t bytes = 0;

    int init(const mxb_grid& g, int device);
    void release();
    int spectra_from_packed_dev(const double* P, cudaStream_t st);
    int spectra_x_component(const double* Pc, int c, cudaStream_t st);
    int spectra_yz(cudaStream_t st);
    // ev (optional): 6 events recorded before P1 and after each of the 5 passes
    int field_dev(const double* m, double* h, cudaStream_t st, const int* halt,
                  cudaEvent_t* ev = nullptr);
};

int make_plan(int L, int dev, Plan1D* p, double2** tw_owned);
int launch_rows_r2c(const Plan1D& p, const double* in, long long in_cstride, int in_pitch,
                    int n_in, double2* out, int hxp, int hx, int nc, long long nrows,
                    cudaStream_t st, const int* halt, int ostride = 0, int coff = 0);
int launch_lines(int dir, const Plan1D& p, const double2* in, double2* out, int n_in, int n_out,
                 long long ES_in, long long ES_out, int Q, long long nlines, long long OS_in,
                 long long OS_out, cudaStream_t st, const int* halt);

// GPU Newell tensor builder (newell.cu)
int newell_packed_component(const Grid& g, int comp, int symmetric, double* packed_c,
                            double* lattice_scratch, cudaStream_t st);
int newell_elements(const Grid& g, double* out6, double* lattice_scratch, cudaStream_t st);

}  // namespace mxb
