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
// x rows; spectra row kx lives at X[(kx / CH) * BLKE + (row * CHP + kx % CH) * 3 + c]
// (one block per destination rank of the slab all-to-all; CH >= hx for one rank)
int fast_rows(bool fwd, int M, const double* in_r, double2* X, double* out_r, long long cstride,
              int pitch, int nhalf, int CH, int CHP, long long BLKE, long long nrows,
              const double2* twM, const double2* tw2M, cudaStream_t st, const int* halt);

// warp-FFT x passes for nx = 512 (x_warp.cu); -1 when the shape is not covered
int warp_rows(bool fwd, int M, const double* in_r, double2* X, double* out_r, long long cstride, int pitch,
              int nhalf, int CH, int CHP, long long BLKE, long long nrows, const double2* twM,
              const double2* tw2M, cudaStream_t st, const int* halt);

// L2-resident y/z pipeline over kx planes (yz_pipe.cu)
bool pipe_shape_ok(int ny, int nz);
// hx planes of XP (the rank's kx chunk); slab: XP = [g][hx][nzl][ny][3] blocks of gstride elements
int pipe_yz(double2* XP, double2* slot, const double* Kp, unsigned* bar, int hx, int n, double scale,
            const double2* tw, cudaStream_t st, const int* halt, int cplx, int nzl = 0, long long gstride = 0);
// planes kx0 .. kx0+hx-1 of the full spectra K
int pipe_quarter(const double2* K, double* Kp, int L, int hx, int hxp, cudaStream_t st, int kx0 = 0);
bool pipe_cplx_ok(int L);
int pipe_complex(const double2* K, double2* Kx, int L, int hx, int hxp, cudaStream_t st, int kx0 = 0);
// long y lines (longy.cu)
bool longy_shape_ok(int py);
int longy_rows(int dir, int L, const double2* in, double2* out, int n_in, int n_out, long long rows,
               const double2* tw, cudaStream_t st, const int* halt, int nz = 1, int nzl = 0,
               long long gstride = 0);
int longy_quarter(const double2* K, double* Kp, int py, int pz, int hx, int hxp, cudaStream_t st, int kx0 = 0);
int longy_rm_to_pm(const double2* in, double2* out, int ny, int nz, int hx, int hxp, cudaStream_t st);

struct DemagPlan {
    int dev = 0;
    Grid g{};                // GLOBAL grid
    int px = 1, py = 1, pz = 1, hx = 1, hxp = 8;
    double scale = 1.0;
    Plan1D plx{}, ply{}, plz{};
    double2* tw[3] = {nullptr, nullptr, nullptr};
    // z-slab decomposition (G ranks): the x passes run on this rank's nz_l
    // planes, the y/z passes on its kx chunk [kx0, kx0+kxn) of all nz planes.
    int G = 1, rank = 0, nz_l = 1, z0 = 0;
    int CH = 1, CHP = 8, kx0 = 0, kxn = 1;
    long long blk = 0;       // complex elements per all-to-all block
    long long xblk = 0;      // the x passes' block stride (== blk, except the slab pipeline: one local plane)
    double2* XS = nullptr;   // x-pass side, [G][nz_l][ny][CHP][3] (send layout)
    double2* XR = nullptr;   // kx-chunk side, [nz][ny][CHP][3] (== XS for one rank)
    double2* X2 = nullptr;   // [nz][py][CHP][3]
    double2* K = nullptr;    // spectra build scratch [pz][py][kpitch][6] complex: all hx planes
                             // (one rank) or only this rank's kx chunk (slab: kpitch = CHP)
    int kpitch = 0, koff = 0;   // kx pitch of K and the global kx of its first column
    double2* T = nullptr;    // slab build: one component's full x spectrum [pz][py][hxp]
    double2* Kc = nullptr;   // complex spectra of the chunk [pz][py][CHP][6]
    double* Kq = nullptr;    // parity-reduced real spectra of the chunk [L/2+1][G/2+1][CHP][6]
    int kmode = 0;           // 0 complex Kc, 2 real quarter Kq, 3 plane pipeline Kp, 4 long-y Kp,
                             // 5 plane pipeline with complex spectra (Kp holds [hx][L][L][6] double2)
    // plane pipeline (kmode 3): XS is plane-major [kx][z][y][3] (CH = CHP = 1)
    bool pipe = false;
    bool longy = false;       // plane-major long-y path (longy.cu)
    double* Kp = nullptr;     // [hx][py/2+1][pz/2+1][6]
    double2* slots = nullptr; // 3 x [nz][py][3]
    unsigned* bar = nullptr;
    Plan1D plm{};            // length px/2 (fast x rows)
    double2* twm = nullptr;
    bool fast = true;        // use the register-resident kernels where shapes allow
    bool has_kernel = false;
    size_t bytes = 0;
    int fused_L() const { return pz > 1 ? pz : (py > 1 ? py : 1); }
    int fused_G() const { return pz > 1 ? py : 1; }

    int init(const mxb_grid& g, int device, int nranks = 1, int rank = 0);
    bool pipe_candidate(bool symmetric = true) const;
    bool longy_candidate() const;
    void release();
    int spectra_from_packed_dev(const double* P, cudaStream_t st);
    int spectra_x_component(const double* Pc, int c, cudaStream_t st);
    int spectra_yz(cudaStream_t st);
    int finish_spectra(bool symmetric, cudaStream_t st);   // chunk + optional quarter storage
    // one evaluation (one rank): x forward, y/z, x inverse
    int field_dev(const double* m, double* h, cudaStream_t st, const int* halt,
                  cudaEvent_t* ev = nullptr);
    int x_forward(const double* m_local, cudaStream_t st, const int* halt);
    int yz(cudaStream_t st, const int* halt, cudaEvent_t* ev = nullptr);
    int x_inverse(double* h_local, cudaStream_t st, const int* halt);
    // after a synchronised plane-pipeline evaluation: MXB_ECUDA if its
    // dependency guard fired (the field is then invalid)
    int check_abort();
    // kernels one evaluation launches: x forward, the y/z part, x inverse
    int kernels_per_eval() const { return pipe ? 3 : longy ? 6 : (pz > 1 && py > 1 ? 5 : 3); }
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
int direct_sum(const Grid& g, const double* n6, const double* m, double* h, cudaStream_t st);

}  // namespace mxb
