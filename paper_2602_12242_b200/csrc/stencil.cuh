#pragma once

#include "common.cuh"

namespace mxb {

// What the fused stage kernel does with the torque k = dM/dt of the stage state.
enum StageMode : int {
    M_HEFF = 0,    // out = H_eff                         (h_total_quiet, llg.py:193)
    M_RHS = 1,     // out = dM/dt                         (rhs_total, llg.py:179)
    M_RK1 = 2,     // K1 = k;     out = post(y + c k)     (integrators.py:51-54)
    M_RK2 = 3,     // S  = k;     out = post(y + c k)     (integrators.py:55-58)
    M_RK3 = 4,     // S += k;     out = post(y + c k)     (integrators.py:59-62)
    M_RK4 = 5,     // out = renorm(y + dt/6 (K1 + 2 S + k)) + drift + <m>   (integrators.py:63-64, llg.py:347-362)
    M_EULER = 6,   // out = renorm(y + dt k) + drift + <m>                  (integrators.py:43-45)
};

// Uniform-material constants derived on the host with the reference's
// operation order (fields.py:95-99,71-77; grid.py:228; llg.py:66,72).
struct Derived {
    double pref;       // 2/(mu0 Ms^2)
    double pref_dmi;   // pref * D
    double pref_an;    // pref * Ku
    double slope_p;    // A>0 ? -D/(2A) : 0
    double face;       // harmonic face coefficient of two equal cells
    double gl;         // mu0 * gamma/(1+alpha^2)
    double coef;       // gl*alpha/Ms
    double ms2;        // Ms*Ms
    double inv_ms;     // 1/Ms
    double pref_cub;   // -2 Kc1/(mu0 Ms)
    double pref_bdmi;  // -pref * Db
    double slope_b;    // A>0 ? Db/(2A) : 0
};

struct StageArgs {
    Grid g;
    MatDev mat;
    Derived dv;
    uint32_t terms;
    int ghost;
    int prec, damp;
    int renorm;
    const double* ys;       // stage state (stencil input)
    const double* y;        // step start state
    const double* hd;       // demag field of ys or null
    const double* k1;       // K1 buffer
    double* s;              // S buffer
    const double* bias_field;
    double bias[3];
    double* out;
    double* k1_out;
    double c;               // stage coefficient (dt/2 or dt)
    double dt6;             // dt/6
    Ctl* ctl;
    double* partials;
    const int* halt;
    // z-slab decomposition: neighbour planes of the first/last local plane,
    // (3, ny, nx) each, plus the neighbours' Ms and A for per-cell materials
    const double* halo_lo;
    const double* halo_hi;
    const double* hms_lo;
    const double* hms_hi;
    const double* hA_lo;
    const double* hA_hi;
    int nparts;             // block partials written by the last final-stage kernel (0: one per 256 cells)
};

int launch_stage(int mode, bool exact, const StageArgs& a, cudaStream_t st, bool finalize = true);
// out = base + sum_i c[i] * x[i] (i < n <= 4), optionally renormalised
struct CombArgs {
    double* out;
    const double* base;
    const double* x[4];
    double c[4];
    int n;
    int renorm;
};
int launch_comb(bool exact, const StageArgs& a, const CombArgs& cb, cudaStream_t st);
int launch_final_state(bool exact, const StageArgs& a, const double* vin, double* out,
                       cudaStream_t st);
int launch_term(uint32_t term, int ghost, bool exact, const StageArgs& a, cudaStream_t st);
int launch_renorm(const StageArgs& a, double* m, cudaStream_t st);
int launch_mean(const StageArgs& a, const double* m, cudaStream_t st);
int launch_energies(bool exact, const StageArgs& a, const double* m, const double* hd,
                    cudaStream_t st);
int stage_blocks(long long N);
int launch_finalize(const StageArgs& a, int mode, cudaStream_t st);
int stage_nparts(const StageArgs& a);   // block partials a final-stage launch with these args writes
int launch_partials(const StageArgs& a, double* out8, cudaStream_t st);
int launch_commit(const StageArgs& a, const double* totals8, cudaStream_t st);
Derived derive(const MatDev& m, const Grid& g);

// x-row fused stage (stencil.cu k_stage_x): x c2r of the plane-major demag
// spectra X -> stage update -> x r2c of the new state back into X (stages
// 1-3), single rank, nx = 512.  X is [kx][row][3] with kx planes blke complex
// elements apart; tw512 / tw1024 the length-512 / 1024 twiddle tables.
struct XStage {
    double2* X;
    long long blke;
    const double2* tw512;
    const double2* tw1024;
};
bool xstage_eligible(const StageArgs& a);
int launch_xstage(int mode, bool exact, const StageArgs& a, const XStage& x, cudaStream_t st);

}  // namespace mxb
