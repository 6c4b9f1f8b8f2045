// Fused local effective field + LLG torque + RK4/Euler stage update.
//
// One thread per cell.  Per cell it evaluates, in the reference accumulation
// order (llg.py:112-125,170-175):
//   exchange   flux form with harmonic face A and _StencilPlan ghosts   (fields.py:112-127)
//   anisotropy (2Ku/mu0Ms^2)(M.eK)eK                                    (fields.py:161-163)
//   cubic      [unpinned extension]
//   dmi        interfacial, central differences with DMI-tilt ghosts     (fields.py:142-151)
//   bulk dmi   [unpinned extension]
//   demag      precomputed H_d of this stage state (demag.cu)
//   bias       uniform vector at the stage time and/or a spatial field   (llg.py:162-164)
// then the torque (llg.py:64-74) and the integrator stage (integrators.py:43-64),
// with the renormalisation hook (grid.py:178-200), the pre-renormalisation
// blow-up drift and <m> (llg.py:347-362) reduced deterministically.
//
// EXACT=true follows numpy's per-operation rounding (no FMA, true divisions),
// which makes the local terms bit-identical to the reference; EXACT=false
// lets nvcc contract and replaces constant divisions by reciprocal products.
#include <float.h>
#include <limits.h>

#include <stdlib.h>

#include <algorithm>

#include "fft_warp.cuh"
#include "stencil.cuh"
#include "tma.cuh"

namespace mxb {

static const int kBlock = 256;

int stage_blocks(long long N) {
    const long long nb = (N + kBlock - 1) / kBlock;
    return (int)std::max<long long>(nb, 1);
}

__global__ void k_finalize(Ctl* ctl, const double* partials, int nblk, int mode, const int* halt);
__global__ void k_partials(const Ctl* ctl, const double* partials, int nblk, double* out8);
__global__ void k_commit(Ctl* ctl, const double* totals8);

// slab decomposition: local (sum m/Ms x3 | drift, halt, -dead) of the last final stage
int launch_partials(const StageArgs& a, double* out8, cudaStream_t st) {
    k_partials<<<1, 1024, 0, st>>>(a.ctl, a.partials, a.nparts > 0 ? a.nparts : stage_blocks(a.g.N), out8);
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

int launch_commit(const StageArgs& a, const double* totals8, cudaStream_t st) {
    k_commit<<<1, 32, 0, st>>>(a.ctl, totals8);
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

int launch_finalize(const StageArgs& a, int mode, cudaStream_t st) {
    k_finalize<<<1, 1024, 0, st>>>(a.ctl, a.partials, a.nparts > 0 ? a.nparts : stage_blocks(a.g.N),
                                   mode, a.halt);
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

Derived derive(const MatDev& m, const Grid& g) {
    // evaluated with plain IEEE double ops (compiled with -ffp-contract=off)
    Derived d{};
    const double mu0 = MXB_MU0;
    const bool mag = m.Ms > 0.0;
    d.pref = mag ? 2.0 / (mu0 * (m.Ms * m.Ms)) : 0.0;
    d.pref_dmi = d.pref * m.D;
    d.pref_an = d.pref * m.Ku;
    d.slope_p = m.A > 0.0 ? -m.D / (2.0 * m.A) : 0.0;
    const double tot = m.A + m.A;
    d.face = tot > 0.0 ? 2.0 * m.A * m.A / tot : 0.0;
    d.gl = mu0 * (m.gamma / (1.0 + m.alpha * m.alpha));
    d.coef = mag ? d.gl * m.alpha / m.Ms : 0.0;
    d.ms2 = m.Ms * m.Ms;
    d.inv_ms = mag ? 1.0 / m.Ms : 0.0;
    d.pref_cub = mag ? -2.0 * m.Kc1 / (mu0 * m.Ms) : 0.0;
    d.pref_bdmi = -d.pref * m.Db;
    d.slope_b = m.A > 0.0 ? m.Db / (2.0 * m.A) : 0.0;
    (void)g;
    return d;
}

// ---------------------------------------------------------------------------
// per-cell material
// ---------------------------------------------------------------------------
struct CellMat {
    double Ms, A, Ku, D, alpha, ek0, ek1, ek2, Kc1, Db;
    bool mag;
    double pref, pref_dmi, pref_an, slope_p, gl, coef, ms2;
};

template <bool E, bool U>
__device__ __forceinline__ CellMat cell_mat(const StageArgs& a, long long idx) {
    CellMat c;
    const MatDev& m = a.mat;
    const long long N = a.g.N;
    if (U) {
        c.Ms = m.Ms; c.A = m.A; c.Ku = m.Ku; c.D = m.D; c.alpha = m.alpha;
        c.ek0 = m.ek[0]; c.ek1 = m.ek[1]; c.ek2 = m.ek[2];
        c.Kc1 = m.Kc1; c.Db = m.Db;
        c.mag = m.Ms > 0.0;
        c.pref = a.dv.pref; c.pref_dmi = a.dv.pref_dmi; c.pref_an = a.dv.pref_an;
        c.slope_p = a.dv.slope_p; c.gl = a.dv.gl; c.coef = a.dv.coef; c.ms2 = a.dv.ms2;
        return c;
    }
    c.Ms = m.Ms_c ? m.Ms_c[idx] : m.Ms;
    c.A = m.A_c ? m.A_c[idx] : m.A;
    c.Ku = m.Ku_c ? m.Ku_c[idx] : m.Ku;
    c.D = m.D_c ? m.D_c[idx] : m.D;
    c.alpha = m.alpha_c ? m.alpha_c[idx] : m.alpha;
    if (m.ek_c) { c.ek0 = m.ek_c[idx]; c.ek1 = m.ek_c[N + idx]; c.ek2 = m.ek_c[2 * N + idx]; }
    else { c.ek0 = m.ek[0]; c.ek1 = m.ek[1]; c.ek2 = m.ek[2]; }
    c.Kc1 = m.Kc1; c.Db = m.Db;
    c.mag = c.Ms > 0.0;
    c.ms2 = mul<E>(c.Ms, c.Ms);
    c.pref = c.mag ? div_rn(2.0, mul<E>(MXB_MU0, c.ms2)) : 0.0;
    c.pref_dmi = mul<E>(c.pref, c.D);
    c.pref_an = mul<E>(c.pref, c.Ku);
    c.slope_p = c.A > 0.0 ? div_rn(-c.D, mul<E>(2.0, c.A)) : 0.0;
    c.gl = mul<E>(MXB_MU0, div_rn(m.gamma, add<E>(1.0, mul<E>(c.alpha, c.alpha))));
    c.coef = c.mag ? div_rn(mul<E>(c.gl, c.alpha), c.Ms) : 0.0;
    return c;
}

__device__ __forceinline__ double ld(const double* p, long long i) { return __ldg(p + i); }

// Neighbour of cell idx along `axis` (0 x, 1 y, 2 z) in direction `step`,
// exactly as _StencilPlan.neighbor + a_face (fields.py:59-92).
template <bool E, bool U>
__device__ __forceinline__ void neighbour(const StageArgs& a, const double* f, long long idx,
                                          int coord, int n, long long stride, int step, int axis,
                                          const double m[3], const CellMat& cm, double nb[3],
                                          double& face) {
    const long long N = a.g.N;
    const bool periodic = a.ghost == MXB_GHOST_PERIODIC;
    const int c2 = coord + step;
    const bool inr = c2 >= 0 && c2 < n;
    if (axis == 2 && !inr && (c2 < 0 ? a.halo_lo : a.halo_hi)) {
        // neighbour plane owned by the adjacent z-slab
        const bool lo = c2 < 0;
        const double* hp = lo ? a.halo_lo : a.halo_hi;
        const long long plane = (long long)a.g.nx * a.g.ny;
        const long long p = idx - (long long)coord * plane;
        bool valid;
        double Anb;
        if (U) {
            valid = cm.mag;
            Anb = cm.A;
        } else {
            const double* hm = lo ? a.hms_lo : a.hms_hi;
            const double* ha = lo ? a.hA_lo : a.hA_hi;
            valid = (hm ? hm[p] : a.mat.Ms) > 0.0;
            Anb = ha ? ha[p] : a.mat.A;
        }
        double harm;
        if (U) {
            harm = a.dv.face;
        } else {
            const double tot = add<E>(cm.A, Anb);
            harm = tot > 0.0 ? div_rn(mul<E>(mul<E>(2.0, cm.A), Anb), tot) : 0.0;
        }
        face = valid ? harm : cm.A;
        if (periodic || valid) {
            nb[0] = ld(hp, p); nb[1] = ld(hp, plane + p); nb[2] = ld(hp, 2 * plane + p);
        } else {
            nb[0] = m[0]; nb[1] = m[1]; nb[2] = m[2];   // z faces carry no DMI tilt
        }
        return;
    }
    long long nidx;
    if (periodic) {
        const int w = inr ? c2 : (c2 < 0 ? c2 + n : c2 - n);
        nidx = idx + (long long)(w - coord) * stride;
    } else {
        nidx = inr ? idx + step * stride : idx;
    }
    bool valid;
    double Anb;
    if (U) {
        valid = (periodic || inr) && cm.mag;
        Anb = cm.A;
    } else {
        const double msn = a.mat.Ms_c ? ld(a.mat.Ms_c, nidx) : a.mat.Ms;
        valid = (periodic || inr) && msn > 0.0;
        Anb = a.mat.A_c ? ld(a.mat.A_c, nidx) : a.mat.A;
    }
    double harm;
    if (U) {
        harm = a.dv.face;
    } else {
        const double tot = add<E>(cm.A, Anb);
        harm = tot > 0.0 ? div_rn(mul<E>(mul<E>(2.0, cm.A), Anb), tot) : 0.0;
    }
    face = valid ? harm : cm.A;
    if (periodic || valid) {
        nb[0] = ld(f, nidx);
        nb[1] = ld(f, N + nidx);
        nb[2] = ld(f, 2 * N + nidx);
    } else if (a.ghost == MXB_GHOST_NEUMANN) {
        nb[0] = m[0]; nb[1] = m[1]; nb[2] = m[2];
    } else {
        // DMI tilt: M + (step*d) * slope (grid.py:217-235)
        const double d = axis == 0 ? a.g.dx : (axis == 1 ? a.g.dy : a.g.dz);
        const double sd = step > 0 ? d : -d;
        const double p = cm.slope_p;
        if (axis == 0) {
            nb[0] = add<E>(m[0], mul<E>(sd, mul<E>(p, m[2])));
            nb[1] = add<E>(m[1], mul<E>(sd, 0.0));
            nb[2] = add<E>(m[2], mul<E>(sd, mul<E>(-p, m[0])));
        } else if (axis == 1) {
            nb[0] = add<E>(m[0], mul<E>(sd, 0.0));
            nb[1] = add<E>(m[1], mul<E>(sd, mul<E>(p, m[2])));
            nb[2] = add<E>(m[2], mul<E>(sd, mul<E>(-p, m[1])));
        } else {
            nb[0] = m[0]; nb[1] = m[1]; nb[2] = m[2];
        }
    }
}

// bulk-DMI neighbour: raw neighbour if in range and magnetic, else the
// natural-boundary ghost M + step*d*(Db/2A)(e_k x M)   [unpinned extension]
template <bool U>
__device__ __forceinline__ void bulk_neighbour(const StageArgs& a, const double* f, long long idx,
                                               int coord, int n, long long stride, int step,
                                               int axis, const double m[3], const CellMat& cm,
                                               double nb[3]) {
    const long long N = a.g.N;
    const int c2 = coord + step;
    if (axis == 2 && (c2 < 0 ? a.halo_lo : (c2 >= n ? a.halo_hi : nullptr))) {
        const bool lo = c2 < 0;
        const double* hp = lo ? a.halo_lo : a.halo_hi;
        const long long plane = (long long)a.g.nx * a.g.ny;
        const long long p = idx - (long long)coord * plane;
        const double* hm = lo ? a.hms_lo : a.hms_hi;
        if (U || !hm || hm[p] > 0.0) {
            nb[0] = ld(hp, p); nb[1] = ld(hp, plane + p); nb[2] = ld(hp, 2 * plane + p);
            return;
        }
    }
    bool valid = c2 >= 0 && c2 < n;
    const long long nidx = valid ? idx + step * stride : idx;
    if (valid && !U && a.mat.Ms_c) valid = ld(a.mat.Ms_c, nidx) > 0.0;
    if (valid) {
        nb[0] = ld(f, nidx); nb[1] = ld(f, N + nidx); nb[2] = ld(f, 2 * N + nidx);
        return;
    }
    const double d = axis == 0 ? a.g.dx : (axis == 1 ? a.g.dy : a.g.dz);
    const double sd = step > 0 ? d : -d;
    const double pr = U ? a.dv.slope_b : (cm.A > 0.0 ? cm.Db / (2.0 * cm.A) : 0.0);
    double cr[3];
    if (axis == 0) { cr[0] = 0.0; cr[1] = -m[2]; cr[2] = m[1]; }
    else if (axis == 1) { cr[0] = m[2]; cr[1] = 0.0; cr[2] = -m[0]; }
    else { cr[0] = -m[1]; cr[1] = m[0]; cr[2] = 0.0; }
    for (int q = 0; q < 3; ++q) nb[q] = m[q] + sd * (pr * cr[q]);
}

template <bool E, bool U>
__device__ __forceinline__ void heff_nb(const StageArgs& a, const double* f, long long idx, int i,
                                        int j, int k, const double m[3], const CellMat& cm,
                                        uint32_t terms, const double xp[3], const double xm[3],
                                        const double yp[3], const double ym[3], const double zp[3],
                                        const double zm[3], double fxp, double fxm, double fyp,
                                        double fym, double fzp, double fzm, double h[3],
                                        const double* hd_pre = nullptr);

// H_eff of one cell in the reference accumulation order.
template <bool E, bool U>
__device__ __forceinline__ void heff_cell(const StageArgs& a, const double* f, long long idx, int i,
                                          int j, int k, const double m[3], const CellMat& cm,
                                          uint32_t terms, double h[3]) {
    const Grid& g = a.g;
    h[0] = 0.0; h[1] = 0.0; h[2] = 0.0;
    const bool ex = terms & MXB_TERM_EXCHANGE;
    const bool dmi = terms & MXB_TERM_DMI;
    double xp[3], xm[3], yp[3], ym[3], zp[3], zm[3];
    double fxp = 0, fxm = 0, fyp = 0, fym = 0, fzp = 0, fzm = 0;
    const bool need_x = (ex && g.nx > 1) || dmi;
    const bool need_y = (ex && g.ny > 1) || dmi;
    const bool need_z = ex && g.nz > 1;
    const long long sy = g.nx, sz = (long long)g.nx * g.ny;
    if (need_x) {
        neighbour<E, U>(a, f, idx, i, g.nx, 1, +1, 0, m, cm, xp, fxp);
        neighbour<E, U>(a, f, idx, i, g.nx, 1, -1, 0, m, cm, xm, fxm);
    }
    if (need_y) {
        neighbour<E, U>(a, f, idx, j, g.ny, sy, +1, 1, m, cm, yp, fyp);
        neighbour<E, U>(a, f, idx, j, g.ny, sy, -1, 1, m, cm, ym, fym);
    }
    if (need_z) {
        neighbour<E, U>(a, f, idx, k, g.nz, sz, +1, 2, m, cm, zp, fzp);
        neighbour<E, U>(a, f, idx, k, g.nz, sz, -1, 2, m, cm, zm, fzm);
    }
    heff_nb<E, U>(a, f, idx, i, j, k, m, cm, terms, xp, xm, yp, ym, zp, zm, fxp, fxm, fyp, fym, fzp,
                  fzm, h);
}

// H_eff from gathered neighbours (values after the ghost rules) and face
// coefficients, in the reference accumulation order.
template <bool E, bool U>
__device__ __forceinline__ void heff_nb(const StageArgs& a, const double* f, long long idx, int i,
                                        int j, int k, const double m[3], const CellMat& cm,
                                        uint32_t terms, const double xp[3], const double xm[3],
                                        const double yp[3], const double ym[3], const double zp[3],
                                        const double zm[3], double fxp, double fxm, double fyp,
                                        double fym, double fzp, double fzm, double h[3],
                                        const double* hd_pre) {
    const Grid& g = a.g;
    h[0] = 0.0; h[1] = 0.0; h[2] = 0.0;
    const bool ex = terms & MXB_TERM_EXCHANGE;
    const bool dmi = terms & MXB_TERM_DMI;
    const long long sy = g.nx, sz = (long long)g.nx * g.ny;
    if (ex) {
        double acc[3] = {0.0, 0.0, 0.0};
        if (g.nx > 1) {
            const double dd = mul<E>(g.dx, g.dx);
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const double t = sub<E>(mul<E>(fxp, sub<E>(xp[q], m[q])), mul<E>(fxm, sub<E>(m[q], xm[q])));
                acc[q] = add<E>(acc[q], E ? div_rn(t, dd) : t * (1.0 / dd));
            }
        }
        if (g.ny > 1) {
            const double dd = mul<E>(g.dy, g.dy);
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const double t = sub<E>(mul<E>(fyp, sub<E>(yp[q], m[q])), mul<E>(fym, sub<E>(m[q], ym[q])));
                acc[q] = add<E>(acc[q], E ? div_rn(t, dd) : t * (1.0 / dd));
            }
        }
        if (g.nz > 1) {
            const double dd = mul<E>(g.dz, g.dz);
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const double t = sub<E>(mul<E>(fzp, sub<E>(zp[q], m[q])), mul<E>(fzm, sub<E>(m[q], zm[q])));
                acc[q] = add<E>(acc[q], E ? div_rn(t, dd) : t * (1.0 / dd));
            }
        }
        if (cm.mag) {
#pragma unroll
            for (int q = 0; q < 3; ++q) h[q] = add<E>(h[q], mul<E>(cm.pref, acc[q]));
        }
    }
    if (terms & MXB_TERM_ANISOTROPY) {
        const double proj = add<E>(add<E>(mul<E>(m[0], cm.ek0), mul<E>(m[1], cm.ek1)), mul<E>(m[2], cm.ek2));
        const double t = mul<E>(cm.pref_an, proj);
        h[0] = add<E>(h[0], mul<E>(t, cm.ek0));
        h[1] = add<E>(h[1], mul<E>(t, cm.ek1));
        h[2] = add<E>(h[2], mul<E>(t, cm.ek2));
    }
    if ((terms & MXB_TERM_CUBIC) && cm.mag) {
        const MatDev& mt = a.mat;
        const double inv = 1.0 / cm.Ms;
        const double mn0 = m[0] * inv, mn1 = m[1] * inv, mn2 = m[2] * inv;
        const double a1 = mt.c1[0] * mn0 + mt.c1[1] * mn1 + mt.c1[2] * mn2;
        const double a2 = mt.c2[0] * mn0 + mt.c2[1] * mn1 + mt.c2[2] * mn2;
        const double a3 = mt.c3[0] * mn0 + mt.c3[1] * mn1 + mt.c3[2] * mn2;
        const double p = U ? a.dv.pref_cub : -2.0 * cm.Kc1 / (MXB_MU0 * cm.Ms);
        const double w1 = p * a1 * (a2 * a2 + a3 * a3);
        const double w2 = p * a2 * (a3 * a3 + a1 * a1);
        const double w3 = p * a3 * (a1 * a1 + a2 * a2);
#pragma unroll
        for (int q = 0; q < 3; ++q) h[q] += w1 * mt.c1[q] + w2 * mt.c2[q] + w3 * mt.c3[q];
    }
    if (dmi) {
        const double i2x = 2 * g.dx, i2y = 2 * g.dy;
        const double gx0 = E ? div_rn(sub<E>(xp[0], xm[0]), i2x) : (xp[0] - xm[0]) * (1.0 / i2x);
        const double gx2 = E ? div_rn(sub<E>(xp[2], xm[2]), i2x) : (xp[2] - xm[2]) * (1.0 / i2x);
        const double gy1 = E ? div_rn(sub<E>(yp[1], ym[1]), i2y) : (yp[1] - ym[1]) * (1.0 / i2y);
        const double gy2 = E ? div_rn(sub<E>(yp[2], ym[2]), i2y) : (yp[2] - ym[2]) * (1.0 / i2y);
        if (cm.mag) {
            h[0] = add<E>(h[0], mul<E>(cm.pref_dmi, gx2));
            h[1] = add<E>(h[1], mul<E>(cm.pref_dmi, gy2));
            h[2] = add<E>(h[2], mul<E>(-cm.pref_dmi, add<E>(gx0, gy1)));
        }
    }
    if ((terms & MXB_TERM_BULK_DMI) && cm.mag) {
        double bp[3], bm[3], gr[3][3];
        const int coords[3] = {i, j, k};
        const int ns[3] = {g.nx, g.ny, g.nz};
        const long long strides[3] = {1, sy, sz};
        const double ds[3] = {g.dx, g.dy, g.dz};
        for (int ax = 0; ax < 3; ++ax) {
            bulk_neighbour<U>(a, f, idx, coords[ax], ns[ax], strides[ax], +1, ax, m, cm, bp);
            bulk_neighbour<U>(a, f, idx, coords[ax], ns[ax], strides[ax], -1, ax, m, cm, bm);
            for (int q = 0; q < 3; ++q) gr[ax][q] = (bp[q] - bm[q]) / (2 * ds[ax]);
        }
        const double cx = gr[1][2] - gr[2][1];
        const double cy = gr[2][0] - gr[0][2];
        const double cz = gr[0][1] - gr[1][0];
        const double p = U ? a.dv.pref_bdmi : -(cm.pref * cm.Db);
        h[0] += p * cx; h[1] += p * cy; h[2] += p * cz;
    }
    if (terms & MXB_TERM_DEMAG) {
        const long long N = g.N;
        h[0] = add<E>(h[0], hd_pre ? hd_pre[0] : ld(a.hd, idx));
        h[1] = add<E>(h[1], hd_pre ? hd_pre[1] : ld(a.hd, N + idx));
        h[2] = add<E>(h[2], hd_pre ? hd_pre[2] : ld(a.hd, 2 * N + idx));
    }
    if (terms & MXB_TERM_BIAS) {
        double b0 = a.bias[0], b1 = a.bias[1], b2 = a.bias[2];
        if (a.bias_field) {
            const long long N = g.N;
            b0 = ld(a.bias_field, idx); b1 = ld(a.bias_field, N + idx); b2 = ld(a.bias_field, 2 * N + idx);
        }
        h[0] = add<E>(h[0], b0);
        h[1] = add<E>(h[1], b1);
        h[2] = add<E>(h[2], b2);
    }
}

template <bool E>
__device__ __forceinline__ void torque(const double m[3], const double h[3], const CellMat& cm,
                                       int prec, int damp, double k[3]) {
    const double x0 = sub<E>(mul<E>(m[1], h[2]), mul<E>(m[2], h[1]));
    const double x1 = sub<E>(mul<E>(m[2], h[0]), mul<E>(m[0], h[2]));
    const double x2 = sub<E>(mul<E>(m[0], h[1]), mul<E>(m[1], h[0]));
    k[0] = 0.0; k[1] = 0.0; k[2] = 0.0;
    if (prec) {
        k[0] = add<E>(k[0], mul<E>(cm.gl, x0));
        k[1] = add<E>(k[1], mul<E>(cm.gl, x1));
        k[2] = add<E>(k[2], mul<E>(cm.gl, x2));
    }
    if (damp) {
        const double y0 = sub<E>(mul<E>(m[1], x2), mul<E>(m[2], x1));
        const double y1 = sub<E>(mul<E>(m[2], x0), mul<E>(m[0], x2));
        const double y2 = sub<E>(mul<E>(m[0], x1), mul<E>(m[1], x0));
        k[0] = add<E>(k[0], mul<E>(cm.coef, y0));
        k[1] = add<E>(k[1], mul<E>(cm.coef, y1));
        k[2] = add<E>(k[2], mul<E>(cm.coef, y2));
    }
}

// renormalize one cell (grid.py:184-200); returns false on a dead magnetic cell
template <bool E>
__device__ __forceinline__ bool renorm_cell(double v[3], const CellMat& cm) {
    const double n2 = add<E>(add<E>(mul<E>(v[0], v[0]), mul<E>(v[1], v[1])), mul<E>(v[2], v[2]));
    if (cm.mag && n2 == 0.0) return false;
    const bool stale = cm.mag && fabs(sub<E>(n2, cm.ms2)) > mul<E>(1e-15, cm.ms2);
    double s = 1.0;
    if (stale) s = E ? div_rn(cm.Ms, sqrt(n2)) : cm.Ms * rsqrt(n2);
    if (!cm.mag) s = 0.0;
    v[0] = mul<E>(v[0], s); v[1] = mul<E>(v[1], s); v[2] = mul<E>(v[2], s);
    return true;
}

__device__ __forceinline__ void flag_dead(Ctl* ctl, long long idx) {
    atomicMin((long long*)&ctl->dead_flat, idx);
    atomicCAS(&ctl->halt, 0, (int)MXB_EDEAD);
}

// ---------------------------------------------------------------------------
// block reductions (deterministic for a fixed launch shape)
// ---------------------------------------------------------------------------
template <int NV>
__device__ __forceinline__ void block_reduce(double v[NV], const bool is_max[NV]) {
    __shared__ double sh[32][NV];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < NV; ++q)
        for (int o = 16; o > 0; o >>= 1) {
            const double w = __shfl_down_sync(0xffffffffu, v[q], o);
            v[q] = is_max[q] ? fmax(v[q], w) : v[q] + w;
        }
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < NV; ++q) sh[wid][q] = v[q];
    __syncthreads();
    const int nw = blockDim.x >> 5;
    if (wid == 0) {
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            v[q] = lane < nw ? sh[lane][q] : (is_max[q] ? -DBL_MAX : 0.0);
            for (int o = 16; o > 0; o >>= 1) {
                const double w = __shfl_down_sync(0xffffffffu, v[q], o);
                v[q] = is_max[q] ? fmax(v[q], w) : v[q] + w;
            }
        }
    }
    __syncthreads();
}

// final reduction of NV partial slots over all blocks, by the last block
template <int NV>
__device__ void reduce_partials(const double* partials, int nblk, const bool is_max[NV],
                                double out[NV]) {
    double v[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) v[q] = is_max[q] ? -DBL_MAX : 0.0;
    for (int b = threadIdx.x; b < nblk; b += blockDim.x) {
        volatile const double* p = partials + (long long)b * kReduceSlots;
#pragma unroll
        for (int q = 0; q < NV; ++q) v[q] = is_max[q] ? fmax(v[q], p[q]) : v[q] + p[q];
    }
    block_reduce<NV>(v, is_max);
#pragma unroll
    for (int q = 0; q < NV; ++q) out[q] = v[q];
}

// torque and the integrator stage of one cell given its H_eff (writes outputs,
// accumulates the step partials for the final RK4 / Euler stage)
template <int MODE, bool E>
__device__ __forceinline__ void stage_tail(const StageArgs& a, long long idx, const CellMat& cm,
                                           const double m[3], const double h[3], double red[4],
                                           const double* y_pre = nullptr, const double* k1_pre = nullptr,
                                           const double* s_pre = nullptr, double* v_ret = nullptr) {
    const long long N = a.g.N;
    constexpr bool kFinal = MODE == M_RK4 || MODE == M_EULER;
        if (MODE == M_HEFF) {
        a.out[idx] = h[0]; a.out[N + idx] = h[1]; a.out[2 * N + idx] = h[2];
    } else {
        double kk[3];
        torque<E>(m, h, cm, a.prec, a.damp, kk);
        if (MODE == M_RHS) {
            a.out[idx] = kk[0]; a.out[N + idx] = kk[1]; a.out[2 * N + idx] = kk[2];
        } else {
            const double y[3] = {y_pre ? y_pre[0] : ld(a.y, idx), y_pre ? y_pre[1] : ld(a.y, N + idx),
                                 y_pre ? y_pre[2] : ld(a.y, 2 * N + idx)};
            double v[3];
            if (MODE == M_RK1 || MODE == M_RK2 || MODE == M_RK3 || MODE == M_EULER) {
#pragma unroll
                for (int q = 0; q < 3; ++q) v[q] = add<E>(y[q], mul<E>(a.c, kk[q]));
                if (MODE == M_RK1) {
                    a.k1_out[idx] = kk[0]; a.k1_out[N + idx] = kk[1]; a.k1_out[2 * N + idx] = kk[2];
                } else if (MODE == M_RK2) {
                    a.s[idx] = kk[0]; a.s[N + idx] = kk[1]; a.s[2 * N + idx] = kk[2];
                } else if (MODE == M_RK3) {
#pragma unroll
                    for (int q = 0; q < 3; ++q) a.s[q * N + idx] = add<E>(s_pre ? s_pre[q] : a.s[q * N + idx], kk[q]);
                }
            } else {  // M_RK4
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    const double k1 = k1_pre ? k1_pre[q] : ld(a.k1, q * N + idx);
                    const double s = s_pre ? s_pre[q] : a.s[q * N + idx];
                    v[q] = add<E>(y[q], mul<E>(a.dt6, add<E>(add<E>(k1, mul<E>(2.0, s)), kk[q])));
                }
            }
            if (kFinal) {
                if (cm.mag) {
                    const double n2 = add<E>(add<E>(mul<E>(v[0], v[0]), mul<E>(v[1], v[1])), mul<E>(v[2], v[2]));
                    double d = fabs(sub<E>(E ? div_rn(sqrt(n2), cm.Ms) : sqrt(n2) * (1.0 / cm.Ms), 1.0));
                    if (!(d == d) || isinf(d)) d = DBL_MAX;  // non-finite drift (llg.py:351)
                    red[3] = fmax(red[3], d);
                }
                // a dead cell here always has drift 1 > 0.1, so the blow-up wins
                // (llg.py:348-355); only record it, never halt mid-kernel
                if (!renorm_cell<E>(v, cm)) atomicMin((long long*)&a.ctl->dead_flat, idx);
                if (cm.mag) {
#pragma unroll
                    for (int q = 0; q < 3; ++q)
                        red[q] += E ? div_rn(v[q], cm.Ms) : v[q] * (1.0 / cm.Ms);
                }
            } else if (a.renorm) {
                if (!renorm_cell<E>(v, cm)) flag_dead(a.ctl, idx);
            }
            a.out[idx] = v[0]; a.out[N + idx] = v[1]; a.out[2 * N + idx] = v[2];
            if (v_ret) { v_ret[0] = v[0]; v_ret[1] = v[1]; v_ret[2] = v[2]; }
        }
    }
}

// ---------------------------------------------------------------------------
// the fused stage kernel
// ---------------------------------------------------------------------------
template <int MODE, bool E, bool U>
__global__ void __launch_bounds__(256, 3) k_stage(StageArgs a) {
    if (a.halt && *(volatile const int*)a.halt) return;
    const Grid& g = a.g;
    const long long N = g.N;
    constexpr bool kFinal = MODE == M_RK4 || MODE == M_EULER;
    double red[4] = {0.0, 0.0, 0.0, 0.0};
    // one cell per thread, blocks in cell order: the z-neighbour planes of the
    // resident window are still in L2 when they are needed
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (idx < N) {
        const int i = (int)(idx % g.nx);
        const long long r = idx / g.nx;
        const int j = (int)(r % g.ny), k = (int)(r / g.ny);
        const CellMat cm = cell_mat<E, U>(a, idx);
        const double m[3] = {ld(a.ys, idx), ld(a.ys, N + idx), ld(a.ys, 2 * N + idx)};
        double h[3];
        heff_cell<E, U>(a, a.ys, idx, i, j, k, m, cm, a.terms, h);
        stage_tail<MODE, E>(a, idx, cm, m, h, red);
    }
    if (kFinal) {
        const bool is_max[4] = {false, false, false, true};
        block_reduce<4>(red, is_max);
        if (threadIdx.x == 0) {
            double* p = a.partials + (long long)blockIdx.x * kReduceSlots;
            p[0] = red[0]; p[1] = red[1]; p[2] = red[2]; p[3] = red[3];
        }
    }
}

__global__ void __launch_bounds__(1024) k_partials(const Ctl* ctl, const double* partials, int nblk,
                                                   double* out8) {
    const bool is_max[4] = {false, false, false, true};
    double tot[4];
    if (ctl->halt) {
        if (threadIdx.x == 0) {
            out8[0] = out8[1] = out8[2] = out8[3] = 0.0;
            out8[4] = 0.0;
            out8[5] = (double)ctl->halt;
            out8[6] = ctl->dead_flat == LLONG_MAX ? -9.0e18 : -(double)ctl->dead_flat;
            out8[7] = 0.0;
        }
        return;
    }
    reduce_partials<4>(partials, nblk, is_max, tot);
    if (threadIdx.x == 0) {
        out8[0] = tot[0]; out8[1] = tot[1]; out8[2] = tot[2]; out8[3] = 0.0;
        out8[4] = tot[3] < 0.0 ? 0.0 : tot[3];
        out8[5] = (double)ctl->halt;
        out8[6] = ctl->dead_flat == LLONG_MAX ? -9.0e18 : -(double)ctl->dead_flat;
        out8[7] = 0.0;
    }
}

// global totals (sums over ranks of [0..3], max over ranks of [4..7]) -> the
// same bookkeeping as k_finalize mode 0, identically on every rank
__global__ void k_commit(Ctl* ctl, const double* t) {
    if (threadIdx.x != 0) return;
    Ctl* c = ctl;
    const int halt = (int)t[5];
    if (halt == MXB_EDEAD || halt == MXB_EBLOWUP) {
        c->halt = halt;
        if (t[6] > -9.0e18) c->dead_flat = (long long)(-t[6]);
        return;
    }
    if (c->halt) return;
    const double drift = t[4];
    if (drift == DBL_MAX || drift > 0.10) {
        c->drift = drift;
        c->halt = MXB_EBLOWUP;
        return;
    }
    const double inv = (double)c->n_magnetic;
    double res = 0.0;
    for (int q = 0; q < 3; ++q) {
        const double mq = t[q] / inv;
        res = fmax(res, fabs(mq - c->prev_mean[q]));
        c->mean[q] = mq;
        c->prev_mean[q] = mq;
    }
    c->residual = res;
    c->drift = drift;
    c->steps_done += 1;
    if (c->eq_tol >= 0.0 && res < c->eq_tol) c->halt = MXB_EQUILIBRATED;
}

// Deterministic final reduction of the per-block partials (fixed order for a
// given grid) and the step bookkeeping of Simulation.run_until (llg.py:347-371):
// blow-up test on the pre-renormalisation drift, <m>, residual, equilibrium.
// mode 0: step, 1: mean of a field, 2: energies.
__global__ void __launch_bounds__(1024) k_finalize(Ctl* ctl, const double* partials, int nblk,
                                                   int mode, const int* halt) {
    if (halt && *(volatile const int*)halt) return;
    const bool is_max[4] = {false, false, false, mode == 0};
    double tot[4];
    reduce_partials<4>(partials, nblk, is_max, tot);
    if (threadIdx.x != 0) return;
    Ctl* c = ctl;
    const double inv = (double)c->n_magnetic;
    if (mode == 1) {
        for (int q = 0; q < 3; ++q) c->mean[q] = tot[q] / inv;
        return;
    }
    if (mode == 2) {
        for (int q = 0; q < 4; ++q) c->energies[q] = tot[q] / inv;
        return;
    }
    const double drift = tot[3] < 0.0 ? 0.0 : tot[3];
    if (drift == DBL_MAX || drift > 0.10) {
        c->drift = drift;
        c->halt = MXB_EBLOWUP;
        return;
    }
    double res = 0.0;
    for (int q = 0; q < 3; ++q) {
        const double mq = tot[q] / inv;
        res = fmax(res, fabs(mq - c->prev_mean[q]));
        c->mean[q] = mq;
        c->prev_mean[q] = mq;
    }
    c->residual = res;
    c->drift = drift;
    c->steps_done += 1;
    if (c->eq_tol >= 0.0 && res < c->eq_tol) c->halt = MXB_EQUILIBRATED;
}

// ---------------------------------------------------------------------------
// z-marching variant for uniform, fully magnetic materials: a CTA owns a
// 32 x 8 column tile and walks ZC planes; x/y neighbours come from a shared
// tile with a one-cell halo ring, z neighbours stay in registers.  Same
// neighbour values, face coefficients and arithmetic as k_stage.
// ---------------------------------------------------------------------------
#ifndef MXB_ZTY   // tile rows: 32 x 4 tiles at 4 CTAs per SM beat 32 x 8 at 2 (12.3 vs 12.9 ms per step)
#define MXB_ZTY 4
#endif
#ifndef MXB_ZC   // z planes per CTA; 512^3 stage time per step (32 x 8 tiles): 8 -> 14.37 ms, 16 -> 13.73,
#define MXB_ZC 64  // 32 -> 13.43, 64 -> 13.35; 32 x 4 tiles: 32 -> 12.45, 64 -> 12.33
#endif
#ifndef MXB_ZT_MINB   // CTAs per SM the TMA z-march is compiled for (register budget)
#define MXB_ZT_MINB (16 / MXB_ZTY)
#endif
#ifndef MXB_ZT_DEEP   // TMA z-march: state 3 / aux 2 planes ahead for stages with <= 2 aux fields
#define MXB_ZT_DEEP 0
#endif
#ifndef MXB_ZT_YDEDUP   // TMA z-march: no step-start-state box when it is the stage state
#define MXB_ZT_YDEDUP 1
#endif
#ifndef MXB_ZM_CTAS
#define MXB_ZM_CTAS 3
#endif
#ifndef MXB_ZM_PRELOAD_Y
#define MXB_ZM_PRELOAD_Y 0
#endif
constexpr int ZTX = 32, ZTY = MXB_ZTY, ZC = MXB_ZC;

template <bool E>
__device__ __forceinline__ void ghost_nb(const StageArgs& a, int axis, int step, const double m[3],
                                         double p, double nb[3]) {
    if (a.ghost == MXB_GHOST_NEUMANN || axis == 2) {
        nb[0] = m[0]; nb[1] = m[1]; nb[2] = m[2];
        return;
    }
    const double d = axis == 0 ? a.g.dx : a.g.dy;
    const double sd = step > 0 ? d : -d;
    if (axis == 0) {
        nb[0] = add<E>(m[0], mul<E>(sd, mul<E>(p, m[2])));
        nb[1] = add<E>(m[1], mul<E>(sd, 0.0));
        nb[2] = add<E>(m[2], mul<E>(sd, mul<E>(-p, m[0])));
    } else {
        nb[0] = add<E>(m[0], mul<E>(sd, 0.0));
        nb[1] = add<E>(m[1], mul<E>(sd, mul<E>(p, m[2])));
        nb[2] = add<E>(m[2], mul<E>(sd, mul<E>(-p, m[1])));
    }
}

template <int MODE, bool E>
__global__ void __launch_bounds__(ZTX * ZTY, MXB_ZM_CTAS) k_stage_zm(StageArgs a) {
    if (a.halt && *(volatile const int*)a.halt) return;
    constexpr bool kFinal = MODE == M_RK4 || MODE == M_EULER;
    __shared__ double tile[3][ZTY + 2][ZTX + 2];
    const Grid& g = a.g;
    const long long N = g.N, plane = (long long)g.nx * g.ny;
    const int tx = threadIdx.x & (ZTX - 1), ty = threadIdx.x / ZTX;
    const int i = blockIdx.x * ZTX + tx, j = blockIdx.y * ZTY + ty;
    const int k0 = blockIdx.z * ZC, k1 = min(k0 + ZC, g.nz);
    const bool in = i < g.nx && j < g.ny;
    const long long col = (long long)j * g.nx + i;
    const CellMat cm = cell_mat<E, true>(a, 0);
    const double* f = a.ys;
    double red[4] = {0.0, 0.0, 0.0, 0.0};
    auto load = [&](int k, double v[3]) -> bool {
        if (!in) return false;
        if (k >= 0 && k < g.nz) {
            const long long o = (long long)k * plane + col;
            v[0] = ld(f, o); v[1] = ld(f, N + o); v[2] = ld(f, 2 * N + o);
            return true;
        }
        const double* hp = k < 0 ? a.halo_lo : a.halo_hi;
        if (!hp) return false;
        v[0] = ld(hp, col); v[1] = ld(hp, plane + col); v[2] = ld(hp, 2 * plane + col);
        return true;
    };
    double zmv[3] = {0, 0, 0}, zcv[3] = {0, 0, 0}, zpv[3] = {0, 0, 0};
    load(k0, zcv);
    bool zm_ok = load(k0 - 1, zmv);
    const bool ex = a.terms & MXB_TERM_EXCHANGE;
    const bool kHd = (a.terms & MXB_TERM_DEMAG) && a.hd;
    constexpr bool kY = MXB_ZM_PRELOAD_Y && MODE >= M_RK1;
    for (int k = k0; k < k1; ++k) {
        const bool zp_ok = load(k + 1, zpv);
        // this plane's demag field (and step-start state) issued before the
        // barriers and the tile fill, so their latency overlaps them
        double hdv[3] = {0.0, 0.0, 0.0}, yv[3] = {0.0, 0.0, 0.0};
        if (in) {
            const long long o = (long long)k * plane + col;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                if (kHd) hdv[q] = ld(a.hd, q * N + o);
                if (kY) yv[q] = ld(a.y, q * N + o);
            }
        }
        __syncthreads();
        if (in) {
            const long long o = (long long)k * plane + col;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                tile[q][ty + 1][tx + 1] = zcv[q];
                if (tx == 0 && i > 0) tile[q][ty + 1][0] = ld(f, q * N + o - 1);
                if (tx == ZTX - 1 && i + 1 < g.nx) tile[q][ty + 1][ZTX + 1] = ld(f, q * N + o + 1);
                if (ty == 0 && j > 0) tile[q][0][tx + 1] = ld(f, q * N + o - g.nx);
                if (ty == ZTY - 1 && j + 1 < g.ny) tile[q][ZTY + 1][tx + 1] = ld(f, q * N + o + g.nx);
            }
        }
        __syncthreads();
        if (in) {
            const long long idx = (long long)k * plane + col;
            const double m[3] = {zcv[0], zcv[1], zcv[2]};
            double xp[3], xm[3], yp[3], ym[3], zp[3], zm[3];
            const double hf = a.dv.face, A = cm.A, p = cm.slope_p;
            const bool okxp = i + 1 < g.nx, okxm = i > 0, okyp = j + 1 < g.ny, okym = j > 0;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                xp[q] = tile[q][ty + 1][tx + 2];
                xm[q] = tile[q][ty + 1][tx];
                yp[q] = tile[q][ty + 2][tx + 1];
                ym[q] = tile[q][ty][tx + 1];
                zp[q] = zpv[q];
                zm[q] = zmv[q];
            }
            if (!okxp) ghost_nb<E>(a, 0, +1, m, p, xp);
            if (!okxm) ghost_nb<E>(a, 0, -1, m, p, xm);
            if (!okyp) ghost_nb<E>(a, 1, +1, m, p, yp);
            if (!okym) ghost_nb<E>(a, 1, -1, m, p, ym);
            if (!zp_ok) ghost_nb<E>(a, 2, +1, m, p, zp);
            if (!zm_ok) ghost_nb<E>(a, 2, -1, m, p, zm);
            double h[3];
            (void)ex;
            heff_nb<E, true>(a, f, idx, i, j, k, m, cm, a.terms, xp, xm, yp, ym, zp, zm,
                             okxp ? hf : A, okxm ? hf : A, okyp ? hf : A, okym ? hf : A,
                             zp_ok ? hf : A, zm_ok ? hf : A, h, kHd ? hdv : nullptr);
            stage_tail<MODE, E>(a, idx, cm, m, h, red, kY ? yv : nullptr);
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) { zmv[q] = zcv[q]; zcv[q] = zpv[q]; }
        zm_ok = true;
    }
    if (kFinal) {
        const bool is_max[4] = {false, false, false, true};
        block_reduce<4>(red, is_max);
        if (threadIdx.x == 0) {
            const long long b = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
            double* pp = a.partials + b * kReduceSlots;
            pp[0] = red[0]; pp[1] = red[1]; pp[2] = red[2]; pp[3] = red[3];
        }
    }
}


// ---------------------------------------------------------------------------
// TMA variant of the z-marching stage kernel (single rank, even nx): the state
// planes (tile + one-cell halo ring, 3 components) arrive as 4-D tensor boxes
// {34, 10, 1, 3} in a four-plane ring, plane k+2 issued at the start of plane
// k; the per-plane inputs the mode reads (demag field, step-start state, K1,
// S) as boxes {32, 8, 1, 3} in a two-plane ring.  All loads complete on
// mbarriers, so nothing is prefetched into registers and the arithmetic is
// that of k_stage_zm (bit-identical results).
// ---------------------------------------------------------------------------
struct ZtMaps {
    CUtensorMap st;                 // ys with halo boxes
    CUtensorMap aux[4];             // hd, y, k1, s (as needed)
};

template <int MODE> struct ZtAux {
    static constexpr bool kY = MODE >= M_RK1, kK1 = MODE == M_RK4, kS = MODE == M_RK3 || MODE == M_RK4;
};

// SD: state planes issued ahead of the one being waited for (ring of SD + 2
// slots: planes k-1, k, k+1 in use), AD: aux planes issued ahead (AD + 1 slots)
template <int MODE, bool E, int SD, int AD>
__global__ void __launch_bounds__(ZTX * ZTY, MXB_ZT_MINB) k_stage_zt(StageArgs a, const __grid_constant__ ZtMaps maps,
                                                            int nfields, int has_hd, int y_is_ys) {
    if (a.halt && *(volatile const int*)a.halt) return;
    constexpr bool kFinal = MODE == M_RK4 || MODE == M_EULER;
    // state box (doubles): the x origin of a TMA box must be 16-byte aligned,
    // so the box starts two cells left of the tile (i0 - 2) and one row above
    constexpr int SX = ZTX + 4, SY = ZTY + 2, SBOX = 3 * SY * SX;
    constexpr int SPL = (SBOX + 15) / 16 * 16;                          // slot stride: 128-byte aligned
    constexpr int APL = 3 * ZTY * ZTX;                              // one aux field plane
    constexpr int NS = SD + 2, NA = AD + 1;
    extern __shared__ __align__(128) double zsm[];
    double* stp = zsm;                       // [NS][3][SY][SX]
    double* aux = zsm + NS * SPL;            // [NA][nfields][3][ZTY][ZTX]
    __shared__ alignas(8) unsigned long long mst[NS], max_[NA];
    const Grid& g = a.g;
    const long long plane = (long long)g.nx * g.ny;
    const int tx = threadIdx.x & (ZTX - 1), ty = threadIdx.x / ZTX;
    const int i0 = blockIdx.x * ZTX, j0 = blockIdx.y * ZTY;
    const int i = i0 + tx, j = j0 + ty;
    const int k0 = blockIdx.z * ZC, k1 = min(k0 + ZC, g.nz);
    const bool in = i < g.nx && j < g.ny;
    const long long col = (long long)j * g.nx + i;
    const CellMat cm = cell_mat<E, true>(a, 0);
    double red[4] = {0.0, 0.0, 0.0, 0.0};
    const unsigned st_bytes = SBOX * 8, aux_bytes = nfields * APL * 8;

    // plane kk's state slot and phase: n = kk - k0 + 1 (plane k0 - 1 is n = 0), slot
    // n % NS, phase (n / NS) & 1; aux: n = kk - k0, slot n % NA
    auto sslot = [&](int kk) { return (kk - k0 + 1) % NS; };
    auto aslot = [&](int kk) { return (kk - k0) % NA; };
    auto issue_state = [&](int kk) {   // thread 0
        unsigned long long* mb = &mst[sslot(kk)];
        mbar_expect(mb, st_bytes);
        tma_load_4d(stp + sslot(kk) * SPL, &maps.st, i0 - 2, j0 - 1, kk, 0, mb);
    };
    auto issue_aux = [&](int kk) {     // thread 0
        unsigned long long* mb = &max_[aslot(kk)];
        mbar_expect(mb, aux_bytes);
        for (int f = 0; f < nfields; ++f)
            tma_load_4d(aux + (aslot(kk) * nfields + f) * APL, &maps.aux[f], i0, j0, kk, 0, mb);
    };
    if (threadIdx.x == 0) {
        for (int q = 0; q < NS; ++q) mbar_init(&mst[q]);
        for (int q = 0; q < NA; ++q) mbar_init(&max_[q]);
        for (int kk = k0 - 1; kk < k0 + SD && kk <= k1; ++kk) issue_state(kk);
        if (nfields)
            for (int kk = k0; kk < k0 + AD && kk < k1; ++kk) issue_aux(kk);
    }
    __syncthreads();
    auto wait_state = [&](int kk) {
        const int n = kk - k0 + 1;
        mbar_wait(&mst[n % NS], (unsigned)(n / NS) & 1u);
    };
    wait_state(k0 - 1);
    wait_state(k0);
    for (int k = k0; k < k1; ++k) {
        if (threadIdx.x == 0) {
            if (k + SD <= k1) issue_state(k + SD);           // slot of plane k - 2
            if (nfields && k + AD < k1) issue_aux(k + AD);   // slot of plane k - 1
        }
        wait_state(k + 1);
        if (nfields) mbar_wait(&max_[aslot(k)], (unsigned)((k - k0) / NA) & 1u);
        if (in) {
            const double* sc = stp + sslot(k) * SPL;
            const double* sp = stp + sslot(k + 1) * SPL;
            const double* sm1 = stp + sslot(k - 1) * SPL;
            auto S = [&](const double* b, int q, int yy, int xx) { return b[(q * SY + yy) * SX + xx]; };
            const long long idx = (long long)k * plane + col;
            double m[3], xp[3], xm[3], yp[3], ym[3], zp[3], zm[3];
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                m[q] = S(sc, q, ty + 1, tx + 2);
                xp[q] = S(sc, q, ty + 1, tx + 3);
                xm[q] = S(sc, q, ty + 1, tx + 1);
                yp[q] = S(sc, q, ty + 2, tx + 2);
                ym[q] = S(sc, q, ty, tx + 2);
                zp[q] = S(sp, q, ty + 1, tx + 2);
                zm[q] = S(sm1, q, ty + 1, tx + 2);
            }
            const bool zp_ok = k + 1 < g.nz, zm_ok = k > 0;
            const double hf = a.dv.face, A = cm.A, p = cm.slope_p;
            const bool okxp = i + 1 < g.nx, okxm = i > 0, okyp = j + 1 < g.ny, okym = j > 0;
            if (!okxp) ghost_nb<E>(a, 0, +1, m, p, xp);
            if (!okxm) ghost_nb<E>(a, 0, -1, m, p, xm);
            if (!okyp) ghost_nb<E>(a, 1, +1, m, p, yp);
            if (!okym) ghost_nb<E>(a, 1, -1, m, p, ym);
            if (!zp_ok) ghost_nb<E>(a, 2, +1, m, p, zp);
            if (!zm_ok) ghost_nb<E>(a, 2, -1, m, p, zm);
            // aux fields in the order hd (if any), y, k1, s
            const double* ab = aux + aslot(k) * nfields * APL;
            double hdv[3], yv[3], k1v[3], sv[3];
            int f = 0;
            auto A3 = [&](int ff, double v[3]) {
#pragma unroll
                for (int q = 0; q < 3; ++q) v[q] = ab[ff * APL + (q * ZTY + ty) * ZTX + tx];
            };
            if (has_hd) A3(f++, hdv);
            if (ZtAux<MODE>::kY) {
                if (y_is_ys) {   // first stage: the step-start state is the stage state (no aux box)
#pragma unroll
                    for (int q = 0; q < 3; ++q) yv[q] = m[q];
                } else {
                    A3(f++, yv);
                }
            }
            if (ZtAux<MODE>::kK1) A3(f++, k1v);
            if (ZtAux<MODE>::kS) A3(f++, sv);
            double h[3];
            heff_nb<E, true>(a, a.ys, idx, i, j, k, m, cm, a.terms, xp, xm, yp, ym, zp, zm,
                             okxp ? hf : A, okxm ? hf : A, okyp ? hf : A, okym ? hf : A,
                             zp_ok ? hf : A, zm_ok ? hf : A, h, has_hd ? hdv : nullptr);
            stage_tail<MODE, E>(a, idx, cm, m, h, red, ZtAux<MODE>::kY ? yv : nullptr,
                                ZtAux<MODE>::kK1 ? k1v : nullptr, ZtAux<MODE>::kS ? sv : nullptr);
        }
        __syncthreads();   // slots of planes k - 1 (state) and k (aux) are reused next
    }
    if (kFinal) {
        const bool is_max[4] = {false, false, false, true};
        block_reduce<4>(red, is_max);
        if (threadIdx.x == 0) {
            const long long b = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
            double* pp = a.partials + b * kReduceSlots;
            pp[0] = red[0]; pp[1] = red[1]; pp[2] = red[2]; pp[3] = red[3];
        }
    }
}

static dim3 zm_grid(const Grid& g) {
    return dim3((g.nx + ZTX - 1) / ZTX, (g.ny + ZTY - 1) / ZTY, (g.nz + ZC - 1) / ZC);
}

// the z-marching kernel needs enough column tiles to fill the GPU (at 32^3 it
// would run 8 CTAs); small grids take the one-cell-per-thread kernel
static bool zm_eligible(const StageArgs& a) {
    static const bool on = getenv("MXB_ZMARCH") == nullptr || atoi(getenv("MXB_ZMARCH")) != 0;
    if (!(on && a.mat.uniform && a.mat.all_magnetic && a.ghost != MXB_GHOST_PERIODIC &&
          !(a.terms & (MXB_TERM_CUBIC | MXB_TERM_BULK_DMI)) && (long long)a.g.nx * a.g.ny >= 256))
        return false;
    const dim3 gz = zm_grid(a.g);
    return (long long)gz.x * gz.y * gz.z >= 4 * 148;
}

int stage_nparts(const StageArgs& a) {
    if (zm_eligible(a)) {
        const dim3 gz = zm_grid(a.g);
        return (int)(gz.x * gz.y * gz.z);
    }
    return stage_blocks(a.g.N);
}

// 4-D float64 map of a (3, nz, ny, nx) field, box {bx, by, 1, 3}
static int field_map(CUtensorMap* tm, const double* f, const Grid& g, unsigned bx, unsigned by) {
    static PFN_cuTensorMapEncodeTiled encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !encode)
            return MXB_ECUDA;
    }
    const cuuint64_t dims[4] = {(cuuint64_t)g.nx, (cuuint64_t)g.ny, (cuuint64_t)g.nz, 3};
    const cuuint64_t strides[3] = {(cuuint64_t)g.nx * 8, (cuuint64_t)g.nx * g.ny * 8, (cuuint64_t)g.N * 8};
    const cuuint32_t box[4] = {bx, by, 1, 3}, estr[4] = {1, 1, 1, 1};
    return encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(f), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS
               ? MXB_OK
               : MXB_ECUDA;
}

template <int MODE, bool E>
static bool launch_zt(const StageArgs& a, cudaStream_t st) {
    const char* ze = getenv("MXB_ZTMA");   // read per launch: tests switch it
    const bool on = !(ze && ze[0] == '0');
    if (!on || a.halo_lo || a.halo_hi || (a.g.nx & 1)) return false;
    ZtMaps mp;
    if (field_map(&mp.st, a.ys, a.g, ZTX + 4, ZTY + 2)) return false;
    int nf = 0;
    const int has_hd = (a.terms & MXB_TERM_DEMAG) && a.hd ? 1 : 0;
    if (has_hd && field_map(&mp.aux[nf++], a.hd, a.g, ZTX, ZTY)) return false;
    // the first stage (and Euler) read the step-start state as the stage state:
    // its values come from the state ring, not a second TMA box of the same data
    const int y_is_ys = MXB_ZT_YDEDUP && a.y == a.ys ? 1 : 0;
    if (ZtAux<MODE>::kY && !y_is_ys && field_map(&mp.aux[nf++], a.y, a.g, ZTX, ZTY)) return false;
    if (ZtAux<MODE>::kK1 && field_map(&mp.aux[nf++], a.k1, a.g, ZTX, ZTY)) return false;
    if (ZtAux<MODE>::kS && field_map(&mp.aux[nf++], a.s, a.g, ZTX, ZTY)) return false;
    // deeper rings for the stages with few aux fields (their bytes in flight per
    // CTA are otherwise the smallest): MXB_ZT_DEEP
    const bool deep = MXB_ZT_DEEP && nf <= 2;
    const int NS = deep ? 5 : 4, NA = deep ? 3 : 2;
    const size_t smem = (size_t)(NS * ((3 * (ZTY + 2) * (ZTX + 4) + 15) / 16 * 16) + NA * nf * 3 * ZTY * ZTX) * sizeof(double);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_stage_zt<MODE, E, 2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
        cudaFuncSetAttribute(k_stage_zt<MODE, E, 3, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
        attr = true;
    }
    if (deep) k_stage_zt<MODE, E, 3, 2><<<zm_grid(a.g), ZTX * ZTY, smem, st>>>(a, mp, nf, has_hd, y_is_ys);
    else k_stage_zt<MODE, E, 2, 1><<<zm_grid(a.g), ZTX * ZTY, smem, st>>>(a, mp, nf, has_hd, y_is_ys);
    return true;
}

template <int MODE>
static void launch_zm(bool exact, const StageArgs& a, cudaStream_t st) {
    if (exact) {
        if (!launch_zt<MODE, true>(a, st)) k_stage_zm<MODE, true><<<zm_grid(a.g), ZTX * ZTY, 0, st>>>(a);
    } else {
        if (!launch_zt<MODE, false>(a, st)) k_stage_zm<MODE, false><<<zm_grid(a.g), ZTX * ZTY, 0, st>>>(a);
    }
}

template <int MODE, bool E>
static void launch_mode_u(const StageArgs& a, cudaStream_t st, int nb) {
    if (a.mat.uniform) k_stage<MODE, E, true><<<nb, kBlock, 0, st>>>(a);
    else k_stage<MODE, E, false><<<nb, kBlock, 0, st>>>(a);
}

template <int MODE>
static void launch_mode(bool exact, const StageArgs& a, cudaStream_t st, int nb) {
    if (exact) launch_mode_u<MODE, true>(a, st, nb);
    else launch_mode_u<MODE, false>(a, st, nb);
}

int launch_stage(int mode, bool exact, const StageArgs& a0, cudaStream_t st, bool finalize) {
    StageArgs a = a0;
    const int nb = stage_blocks(a.g.N);
    if (zm_eligible(a)) {
        const dim3 gz = zm_grid(a.g);
        a.nparts = (int)(gz.x * gz.y * gz.z);
        switch (mode) {
            case M_HEFF: launch_zm<M_HEFF>(exact, a, st); break;
            case M_RHS: launch_zm<M_RHS>(exact, a, st); break;
            case M_RK1: launch_zm<M_RK1>(exact, a, st); break;
            case M_RK2: launch_zm<M_RK2>(exact, a, st); break;
            case M_RK3: launch_zm<M_RK3>(exact, a, st); break;
            case M_RK4: launch_zm<M_RK4>(exact, a, st); break;
            case M_EULER: launch_zm<M_EULER>(exact, a, st); break;
            default: set_error("bad stage mode"); return MXB_EINVAL;
        }
        MXB_LAUNCH_CHECK();
        if (finalize && (mode == M_RK4 || mode == M_EULER)) return launch_finalize(a, 0, st);
        return MXB_OK;
    }
    a.nparts = nb;
    switch (mode) {
        case M_HEFF: launch_mode<M_HEFF>(exact, a, st, nb); break;
        case M_RHS: launch_mode<M_RHS>(exact, a, st, nb); break;
        case M_RK1: launch_mode<M_RK1>(exact, a, st, nb); break;
        case M_RK2: launch_mode<M_RK2>(exact, a, st, nb); break;
        case M_RK3: launch_mode<M_RK3>(exact, a, st, nb); break;
        case M_RK4: launch_mode<M_RK4>(exact, a, st, nb); break;
        case M_EULER: launch_mode<M_EULER>(exact, a, st, nb); break;
        default: set_error("bad stage mode"); return MXB_EINVAL;
    }
    MXB_LAUNCH_CHECK();
    if (finalize && (mode == M_RK4 || mode == M_EULER)) return launch_finalize(a, 0, st);
    return MXB_OK;
}

// a single field term (ExchangeOperator etc.): H of only `term`
int launch_term(uint32_t term, int ghost, bool exact, const StageArgs& a0, cudaStream_t st) {
    StageArgs a = a0;
    a.terms = term;
    a.ghost = ghost;
    return launch_stage(M_HEFF, exact, a, st);
}

// ---------------------------------------------------------------------------
// renormalize / mean / energies
// ---------------------------------------------------------------------------
template <bool U>
__global__ void k_renorm(StageArgs a, double* m) {
    const long long N = a.g.N;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < N;
         idx += (long long)gridDim.x * blockDim.x) {
        const CellMat cm = cell_mat<true, U>(a, idx);
        double v[3] = {m[idx], m[N + idx], m[2 * N + idx]};
        if (!renorm_cell<true>(v, cm)) {
            atomicMin((long long*)&a.ctl->dead_flat, idx);
            continue;
        }
        m[idx] = v[0]; m[N + idx] = v[1]; m[2 * N + idx] = v[2];
    }
}

int launch_renorm(const StageArgs& a, double* m, cudaStream_t st) {
    const int nb = stage_blocks(a.g.N);
    if (a.mat.uniform) k_renorm<true><<<nb, kBlock, 0, st>>>(a, m);
    else k_renorm<false><<<nb, kBlock, 0, st>>>(a, m);
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

// out = base + sum_i c[i] * x[i] (i < n <= 4), then optionally the
// renormalisation hook (grid.py:178-200) -- the stage arithmetic of the
// Knoth-Wolke / multirate steps (integrators.py:67-128)
template <bool E, bool U>
__global__ void __launch_bounds__(256) k_comb(StageArgs a, CombArgs cb) {
    if (a.halt && *(volatile const int*)a.halt) return;
    const long long N = a.g.N;
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (idx >= N) return;
    double v[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        double acc = cb.base ? cb.base[q * N + idx] : 0.0;
        for (int i = 0; i < cb.n; ++i) acc = add<E>(acc, mul<E>(cb.c[i], cb.x[i][q * N + idx]));
        v[q] = acc;
    }
    if (cb.renorm) {
        const CellMat cm = cell_mat<E, U>(a, idx);
        if (!renorm_cell<E>(v, cm)) flag_dead(a.ctl, idx);
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) cb.out[q * N + idx] = v[q];
}

// end of a step computed elsewhere: pre-renormalisation drift, renormalise
// into out, <m> partials (llg.py:347-362); followed by k_finalize(mode 0)
template <bool E, bool U>
__global__ void __launch_bounds__(256) k_final_state(StageArgs a, const double* vin, double* out) {
    if (a.halt && *(volatile const int*)a.halt) return;
    const long long N = a.g.N;
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    double red[4] = {0.0, 0.0, 0.0, 0.0};
    if (idx < N) {
        const CellMat cm = cell_mat<E, U>(a, idx);
        double v[3] = {vin[idx], vin[N + idx], vin[2 * N + idx]};
        if (cm.mag) {
            const double n2 = add<E>(add<E>(mul<E>(v[0], v[0]), mul<E>(v[1], v[1])), mul<E>(v[2], v[2]));
            double d = fabs(sub<E>(E ? div_rn(sqrt(n2), cm.Ms) : sqrt(n2) * (1.0 / cm.Ms), 1.0));
            if (!(d == d) || isinf(d)) d = DBL_MAX;
            red[3] = d;
        }
        if (!renorm_cell<E>(v, cm)) atomicMin((long long*)&a.ctl->dead_flat, idx);
        if (cm.mag)
#pragma unroll
            for (int q = 0; q < 3; ++q) red[q] = E ? div_rn(v[q], cm.Ms) : v[q] * (1.0 / cm.Ms);
        out[idx] = v[0]; out[N + idx] = v[1]; out[2 * N + idx] = v[2];
    }
    const bool is_max[4] = {false, false, false, true};
    block_reduce<4>(red, is_max);
    if (threadIdx.x == 0) {
        double* p = a.partials + (long long)blockIdx.x * kReduceSlots;
        p[0] = red[0]; p[1] = red[1]; p[2] = red[2]; p[3] = red[3];
    }
}

int launch_comb(bool exact, const StageArgs& a, const CombArgs& cb, cudaStream_t st) {
    const int nb = stage_blocks(a.g.N);
    if (exact) {
        if (a.mat.uniform) k_comb<true, true><<<nb, kBlock, 0, st>>>(a, cb);
        else k_comb<true, false><<<nb, kBlock, 0, st>>>(a, cb);
    } else {
        if (a.mat.uniform) k_comb<false, true><<<nb, kBlock, 0, st>>>(a, cb);
        else k_comb<false, false><<<nb, kBlock, 0, st>>>(a, cb);
    }
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

int launch_final_state(bool exact, const StageArgs& a, const double* vin, double* out,
                       cudaStream_t st) {
    const int nb = stage_blocks(a.g.N);
    if (exact) {
        if (a.mat.uniform) k_final_state<true, true><<<nb, kBlock, 0, st>>>(a, vin, out);
        else k_final_state<true, false><<<nb, kBlock, 0, st>>>(a, vin, out);
    } else {
        if (a.mat.uniform) k_final_state<false, true><<<nb, kBlock, 0, st>>>(a, vin, out);
        else k_final_state<false, false><<<nb, kBlock, 0, st>>>(a, vin, out);
    }
    MXB_LAUNCH_CHECK();
    return launch_finalize(a, 0, st);
}

template <bool U>
__global__ void k_mean(StageArgs a, const double* m) {
    const long long N = a.g.N;
    double red[3] = {0.0, 0.0, 0.0};
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < N;
         idx += (long long)gridDim.x * blockDim.x) {
        const CellMat cm = cell_mat<true, U>(a, idx);
        if (!cm.mag) continue;
#pragma unroll
        for (int q = 0; q < 3; ++q) red[q] += div_rn(m[q * N + idx], cm.Ms);
    }
    const bool is_max[3] = {false, false, false};
    block_reduce<3>(red, is_max);
    if (threadIdx.x == 0) {
        double* p = a.partials + (long long)blockIdx.x * kReduceSlots;
        p[0] = red[0]; p[1] = red[1]; p[2] = red[2]; p[3] = 0.0;
    }
}

int launch_mean(const StageArgs& a, const double* m, cudaStream_t st) {
    const int nb = stage_blocks(a.g.N);
    if (a.mat.uniform) k_mean<true><<<nb, kBlock, 0, st>>>(a, m);
    else k_mean<false><<<nb, kBlock, 0, st>>>(a, m);
    MXB_LAUNCH_CHECK();
    StageArgs b = a;
    b.halt = nullptr;
    return launch_finalize(b, 1, st);
}

// energy densities (fields.py:200-242) summed over magnetic cells
template <bool E, bool U>
__global__ void k_energies(StageArgs a, const double* m, const double* hd) {
    const Grid& g = a.g;
    const long long N = g.N;
    double red[4] = {0.0, 0.0, 0.0, 0.0};
    const bool dmi_mode = a.ghost == MXB_GHOST_DMI;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < N;
         idx += (long long)gridDim.x * blockDim.x) {
        const CellMat cm = cell_mat<E, U>(a, idx);
        if (!cm.mag) continue;
        const int i = (int)(idx % g.nx);
        const long long r = idx / g.nx;
        const int j = (int)(r % g.ny), k = (int)(r / g.ny);
        const double mv[3] = {m[idx], m[N + idx], m[2 * N + idx]};
        if (hd) {
            const double dot = add<E>(add<E>(mul<E>(mv[0], hd[idx]), mul<E>(mv[1], hd[N + idx])),
                                      mul<E>(mv[2], hd[2 * N + idx]));
            red[0] += mul<E>(-0.5 * MXB_MU0, dot);
        }
        // normalised m and its neighbours (plan.neighbor on mn)
        const double mn[3] = {div_rn(mv[0], cm.Ms), div_rn(mv[1], cm.Ms), div_rn(mv[2], cm.Ms)};
        double g2 = 0.0;
        const int coords[3] = {i, j, k};
        const int ns[3] = {g.nx, g.ny, g.nz};
        const long long strides[3] = {1, g.nx, (long long)g.nx * g.ny};
        const double ds[3] = {g.dx, g.dy, g.dz};
        for (int ax = 0; ax < 3; ++ax) {
            if (ns[ax] == 1 && !dmi_mode) continue;
            double nb[2][3];
            for (int sgn = 0; sgn < 2; ++sgn) {
                const int step = sgn == 0 ? 1 : -1;
                const bool periodic = a.ghost == MXB_GHOST_PERIODIC;
                const int c2 = coords[ax] + step;
                const bool inr = c2 >= 0 && c2 < ns[ax];
                long long nidx;
                if (periodic) {
                    const int w = inr ? c2 : (c2 < 0 ? c2 + ns[ax] : c2 - ns[ax]);
                    nidx = idx + (long long)(w - coords[ax]) * strides[ax];
                } else {
                    nidx = inr ? idx + step * strides[ax] : idx;
                }
                const double msn = U ? a.mat.Ms : (a.mat.Ms_c ? a.mat.Ms_c[nidx] : a.mat.Ms);
                const bool valid = (periodic || inr) && msn > 0.0;
                if (periodic || valid) {
                    for (int q = 0; q < 3; ++q) nb[sgn][q] = msn > 0.0 ? div_rn(m[q * N + nidx], msn) : 0.0;
                } else if (a.ghost == MXB_GHOST_NEUMANN || ax == 2) {
                    for (int q = 0; q < 3; ++q) nb[sgn][q] = mn[q];
                } else {
                    const double sd = step > 0 ? ds[ax] : -ds[ax];
                    const double p = cm.slope_p;
                    if (ax == 0) {
                        nb[sgn][0] = add<E>(mn[0], mul<E>(sd, mul<E>(p, mn[2])));
                        nb[sgn][1] = add<E>(mn[1], mul<E>(sd, 0.0));
                        nb[sgn][2] = add<E>(mn[2], mul<E>(sd, mul<E>(-p, mn[0])));
                    } else {
                        nb[sgn][0] = add<E>(mn[0], mul<E>(sd, 0.0));
                        nb[sgn][1] = add<E>(mn[1], mul<E>(sd, mul<E>(p, mn[2])));
                        nb[sgn][2] = add<E>(mn[2], mul<E>(sd, mul<E>(-p, mn[1])));
                    }
                }
            }
            const double d2 = 2 * ds[ax];
            const double q0 = div_rn(sub<E>(nb[0][0], nb[1][0]), d2);
            const double q1 = div_rn(sub<E>(nb[0][1], nb[1][1]), d2);
            const double q2 = div_rn(sub<E>(nb[0][2], nb[1][2]), d2);
            g2 = add<E>(g2, add<E>(add<E>(mul<E>(q0, q0), mul<E>(q1, q1)), mul<E>(q2, q2)));
        }
        red[1] += mul<E>(cm.A, g2);
        const double pr = add<E>(add<E>(mul<E>(mn[0], cm.ek0), mul<E>(mn[1], cm.ek1)), mul<E>(mn[2], cm.ek2));
        red[2] += mul<E>(cm.Ku, sub<E>(1.0, mul<E>(pr, pr)));
        if (a.terms & MXB_TERM_BIAS) {
            double b0 = a.bias[0], b1 = a.bias[1], b2 = a.bias[2];
            if (a.bias_field) { b0 = a.bias_field[idx]; b1 = a.bias_field[N + idx]; b2 = a.bias_field[2 * N + idx]; }
            const double dot = add<E>(add<E>(mul<E>(mv[0], b0), mul<E>(mv[1], b1)), mul<E>(mv[2], b2));
            red[3] += mul<E>(-MXB_MU0, dot);
        }
    }
    const bool is_max[4] = {false, false, false, false};
    block_reduce<4>(red, is_max);
    if (threadIdx.x == 0) {
        double* p = a.partials + (long long)blockIdx.x * kReduceSlots;
        p[0] = red[0]; p[1] = red[1]; p[2] = red[2]; p[3] = red[3];
    }
}

int launch_energies(bool exact, const StageArgs& a, const double* m, const double* hd,
                    cudaStream_t st) {
    const int nb = stage_blocks(a.g.N);
    if (exact) {
        if (a.mat.uniform) k_energies<true, true><<<nb, kBlock, 0, st>>>(a, m, hd);
        else k_energies<true, false><<<nb, kBlock, 0, st>>>(a, m, hd);
    } else {
        if (a.mat.uniform) k_energies<false, true><<<nb, kBlock, 0, st>>>(a, m, hd);
        else k_energies<false, false><<<nb, kBlock, 0, st>>>(a, m, hd);
    }
    MXB_LAUNCH_CHECK();
    StageArgs b = a;
    b.halt = nullptr;
    return launch_finalize(b, 2, st);
}

}  // namespace mxb

// ---------------------------------------------------------------------------
// x-row fused stage: the x c2r of the demag spectra, the stage update and (for
// stages 1-3) the x r2c of the new stage state in ONE kernel, for the single-
// rank plane pipeline at nx = 512 (north_star item 3: each stage streams M
// once).  Without it a stage is k_c2r_w (writes H_demag, 24 B/cell), the
// stage kernel (reads it back) and k_r2c_w (reads the new state again):
// 72 B/cell per stage that never leave the SM here.
//
// A CTA is 3 warps and owns a row pair (rows 2b, 2b+1 of the nz*ny x-rows),
// exactly the rows its plane-major spectrum slice X[kx][2b..2b+1][3] holds:
//   1. TMA: the slice (513 x 96 B) into shared memory;
//   2. c2r as k_c2r_w (x_warp.cu), one component per warp; H_demag of the
//      pair stays in the first half of each warp's transpose tile;
//   3. the stage update of the pair's 1024 cells (heff_nb + stage_tail: the
//      arithmetic of k_stage_zt, bit-identical), neighbours read through L1/L2
//      (the y +- 1 rows are the adjacent CTAs', the z +- 1 rows were read
//      ny/2 CTAs earlier and are L2 hits); the new state also goes to the
//      second half of the tiles;
//   4. r2c of the new state as k_r2c_w, and the spectrum slice written back by
//      TMA to the addresses step 1 read (each CTA owns its slice: in place).
// Results are bit-identical to the unfused kernels; the final stage's block
// partials are reduced per row pair.
// ---------------------------------------------------------------------------
#ifndef MXB_XS_PAIR   // k_stage_x: two x-adjacent cells per thread iteration, 16-byte loads
#define MXB_XS_PAIR 0
#endif
#ifndef MXB_XS_SWP   // k_stage_x: next cell's loads issued before this cell's arithmetic
#define MXB_XS_SWP 0
#endif
#ifndef MXB_XS_PREFETCH   // k_stage_x: L2 prefetch of the stage rows during the c2r
#define MXB_XS_PREFETCH 0
#endif

namespace mxb {
namespace {
constexpr int XSM = 512;        // complex FFT length of the x rows (px / 2)
constexpr int XSH = XSM + 1;    // spectrum bins (px / 2 + 1)
}

template <int MODE, bool E, bool R2C>
__global__ void __launch_bounds__(96, 4)
k_stage_x(StageArgs a, const double2* __restrict__ tw512, const double2* __restrict__ tw1024,
          const __grid_constant__ CUtensorMap map_main, const __grid_constant__ CUtensorMap map_tail) {
    if (a.halt && *(volatile const int*)a.halt) return;
    constexpr bool kFinal = MODE == M_RK4;
    constexpr bool kK1 = MODE == M_RK4, kS = MODE == M_RK3 || MODE == M_RK4;
    extern __shared__ __align__(128) double2 S[];
    __shared__ alignas(8) unsigned long long mbar;
    const int c = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long row0 = 2LL * blockIdx.x;
    const int xo0 = (int)(row0 * 6);
    if (threadIdx.x == 0) {
        mbar_init(&mbar);
        mbar_expect(&mbar, XSH * 96);
        tma_load_2d(S, &map_main, xo0, 0, &mbar);
        tma_load_2d(S + 256 * 6, &map_main, xo0, 256, &mbar);
        tma_load_2d(S + 512 * 6, &map_tail, xo0, 512, &mbar);
    }
    __syncthreads();   // mbarrier initialised before anyone polls it
#if MXB_XS_PREFETCH
    if (c == 0 && lane < 18) {
        // the stage phase's rows into L2 while the c2r runs: the state rows
        // r0 - 1 .. r0 + 2 and the pair's z +- 1 rows, and the pair's rows of
        // the step-start state, K1 and S (one bulk prefetch per lane)
        const Grid& g = a.g;
        const long long R = (long long)g.ny * g.nz, N = g.N;
        const int q = lane % 3, kind = lane / 3;
        const double* base = nullptr;
        long long r = row0, nr = 2;
        if (kind == 0) { base = a.ys; r = row0 > 0 ? row0 - 1 : 0; nr = min(row0 + 3, R) - r; }
        else if (kind == 1) { base = a.ys; r = row0 - g.ny; }
        else if (kind == 2) { base = a.ys; r = row0 + g.ny; }
        else if (kind == 3) base = a.y;
        else if (kind == 4 && kK1) base = a.k1;
        else if (kind == 5 && kS) base = a.s;
        if (base && r >= 0 && r + nr <= R) prefetch_l2(base + q * N + r * XSM, (unsigned)(nr * XSM * 8));
    }
#endif
    double2 fa[16], fb[16], v[32];
    {
        double2 twp[16];
#pragma unroll
        for (int m = 0; m < 16; ++m) twp[m] = __ldg(tw1024 + lane + 32 * m);
        mbar_wait(&mbar, 0);
#pragma unroll
        for (int m = 0; m < 16; ++m) {
            const int k = lane + 32 * m;
            const double2 w = twp[m];
#pragma unroll
            for (int ln = 0; ln < 2; ++ln) {
                const double2 xk = S[(k * 2 + ln) * 3 + c];
                const double2 xm = S[((XSM - k) * 2 + ln) * 3 + c];
                const double2 A = make_double2(xk.x + xm.x, xk.y - xm.y);
                const double2 Bm = make_double2(xk.x - xm.x, xk.y + xm.y);
                const double2 B = cmul(Bm, make_double2(w.x, -w.y));
                const double2 z = make_double2(A.x - B.y, A.y + B.x);
                if (ln == 0) fa[m] = z; else fb[m] = z;
            }
        }
    }
    __syncthreads();   // S becomes the transpose tiles
    double2* tile = S + c * 1024;
    fw::fft512x2<1>(fa, fb, v, tile, lane, tw512);
    {
        // H_demag of component c: (x[2n], x[2n+1]) pairs of both lines, first half of the tile
        const int line = lane >> 4, k1 = lane & 15;
        __syncwarp();
#pragma unroll
        for (int k2 = 0; k2 < 16; ++k2) tile[line * 256 + k1 + 16 * k2] = v[fw::p32(k2)];
    }
    __syncthreads();
    // the stage update of the pair's cells
    const Grid& g = a.g;
    const long long N = g.N, plane = (long long)g.nx * g.ny;
    const CellMat cm = cell_mat<E, true>(a, 0);
    const double hf = a.dv.face, Af = cm.A, p = cm.slope_p;
    const double* hd_s = reinterpret_cast<const double*>(S);   // [q][2048]: H_demag at [ln * 512 + x]
    double* out_s = reinterpret_cast<double*>(S) + 1024;       // [q][2048]: new state at [ln * 512 + x]
    double red[4] = {0.0, 0.0, 0.0, 0.0};
    // one cell's inputs (global loads; ghosts applied at compute)
    struct In { double m[3], xp[3], xm[3], yp[3], ym[3], zp[3], zm[3], yv[3], k1v[3], sv[3]; };
    auto load = [&](int e, In& u) {
        const int ln = e >> 9, i = e & (XSM - 1);
        const long long row = row0 + ln;
        const int k = (int)(row / g.ny), j = (int)(row - (long long)k * g.ny);
        const long long idx = row * XSM + i;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const long long o = q * N + idx;
            u.m[q] = ld(a.ys, o);
            u.xp[q] = i + 1 < XSM ? ld(a.ys, o + 1) : 0.0;
            u.xm[q] = i > 0 ? ld(a.ys, o - 1) : 0.0;
            u.yp[q] = j + 1 < g.ny ? ld(a.ys, o + XSM) : 0.0;
            u.ym[q] = j > 0 ? ld(a.ys, o - XSM) : 0.0;
            u.zp[q] = k + 1 < g.nz ? ld(a.ys, o + plane) : 0.0;
            u.zm[q] = k > 0 ? ld(a.ys, o - plane) : 0.0;
            u.yv[q] = ld(a.y, o);
            u.k1v[q] = kK1 ? ld(a.k1, o) : 0.0;
            u.sv[q] = kS ? a.s[o] : 0.0;
        }
    };
    auto cell = [&](int e, In& u) {
        const int ln = e >> 9, i = e & (XSM - 1);
        const long long row = row0 + ln;
        const int k = (int)(row / g.ny), j = (int)(row - (long long)k * g.ny);
        const long long idx = row * XSM + i;
        const bool okxp = i + 1 < XSM, okxm = i > 0, okyp = j + 1 < g.ny, okym = j > 0;
        const bool zp_ok = k + 1 < g.nz, zm_ok = k > 0;
        double hdv[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) hdv[q] = hd_s[q * 2048 + e];
        if (!okxp) ghost_nb<E>(a, 0, +1, u.m, p, u.xp);
        if (!okxm) ghost_nb<E>(a, 0, -1, u.m, p, u.xm);
        if (!okyp) ghost_nb<E>(a, 1, +1, u.m, p, u.yp);
        if (!okym) ghost_nb<E>(a, 1, -1, u.m, p, u.ym);
        if (!zp_ok) ghost_nb<E>(a, 2, +1, u.m, p, u.zp);
        if (!zm_ok) ghost_nb<E>(a, 2, -1, u.m, p, u.zm);
        double h[3], vn[3];
        heff_nb<E, true>(a, a.ys, idx, i, j, k, u.m, cm, a.terms, u.xp, u.xm, u.yp, u.ym, u.zp, u.zm,
                         okxp ? hf : Af, okxm ? hf : Af, okyp ? hf : Af, okym ? hf : Af,
                         zp_ok ? hf : Af, zm_ok ? hf : Af, h, hdv);
        stage_tail<MODE, E>(a, idx, cm, u.m, h, red, u.yv, kK1 ? u.k1v : nullptr, kS ? u.sv : nullptr, vn);
        if (R2C) {
#pragma unroll
            for (int q = 0; q < 3; ++q) out_s[q * 2048 + e] = vn[q];
        }
    };
#if MXB_XS_PAIR
    // two x-adjacent cells per iteration: 16-byte loads of the pair's values (the
    // x neighbours inside the pair come from the pair itself)
    for (int pp = threadIdx.x; pp < XSM; pp += 96) {
        const int e0 = 2 * pp;
        const int ln = e0 >> 9, i0 = e0 & (XSM - 1);
        const long long row = row0 + ln;
        const int k = (int)(row / g.ny), j = (int)(row - (long long)k * g.ny);
        const long long idx0 = row * XSM + i0;
        In u0, u1;
        auto ld2 = [&](const double* b, long long o) {
            return __ldg(reinterpret_cast<const double2*>(b + o));
        };
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const long long o = q * N + idx0;
            const double2 mm = ld2(a.ys, o);
            u0.m[q] = mm.x; u1.m[q] = mm.y;
            u0.xp[q] = mm.y; u1.xm[q] = mm.x;
            u0.xm[q] = i0 > 0 ? ld(a.ys, o - 1) : 0.0;
            u1.xp[q] = i0 + 2 < XSM ? ld(a.ys, o + 2) : 0.0;
            const double2 yp2 = j + 1 < g.ny ? ld2(a.ys, o + XSM) : make_double2(0.0, 0.0);
            const double2 ym2 = j > 0 ? ld2(a.ys, o - XSM) : make_double2(0.0, 0.0);
            const double2 zp2 = k + 1 < g.nz ? ld2(a.ys, o + plane) : make_double2(0.0, 0.0);
            const double2 zm2 = k > 0 ? ld2(a.ys, o - plane) : make_double2(0.0, 0.0);
            const double2 y2 = ld2(a.y, o);
            const double2 k12 = kK1 ? ld2(a.k1, o) : make_double2(0.0, 0.0);
            const double2 s2 = kS ? *reinterpret_cast<const double2*>(a.s + o) : make_double2(0.0, 0.0);
            u0.yp[q] = yp2.x; u1.yp[q] = yp2.y; u0.ym[q] = ym2.x; u1.ym[q] = ym2.y;
            u0.zp[q] = zp2.x; u1.zp[q] = zp2.y; u0.zm[q] = zm2.x; u1.zm[q] = zm2.y;
            u0.yv[q] = y2.x; u1.yv[q] = y2.y; u0.k1v[q] = k12.x; u1.k1v[q] = k12.y;
            u0.sv[q] = s2.x; u1.sv[q] = s2.y;
        }
        cell(e0, u0);
        cell(e0 + 1, u1);
    }
#elif MXB_XS_SWP
    // software pipelined: the next cell's loads are in flight during this cell's arithmetic
    {
        In cur, nxt;
        load(threadIdx.x, cur);
        for (int e = threadIdx.x; e < 2 * XSM; e += 96) {
            if (e + 96 < 2 * XSM) load(e + 96, nxt);
            cell(e, cur);
            cur = nxt;
        }
    }
#else
    for (int e = threadIdx.x; e < 2 * XSM; e += 96) {
        In u;
        load(e, u);
        cell(e, u);
    }
#endif
    if (kFinal) {
        const bool is_max[4] = {false, false, false, true};
        block_reduce<4>(red, is_max);
        if (threadIdx.x == 0) {
            double* pp = a.partials + (long long)blockIdx.x * kReduceSlots;
            pp[0] = red[0]; pp[1] = red[1]; pp[2] = red[2]; pp[3] = red[3];
        }
    }
    if (!R2C) return;
    __syncthreads();   // the new state of the pair is staged
    {
        // packed pairs (x[2n], x[2n+1]) of component c, n < 256 non-zero (k_r2c_w)
        const double2* s0 = tile + 512;
#pragma unroll
        for (int m = 0; m < 16; ++m) {
            fa[m] = m < 8 ? s0[lane + 32 * m] : make_double2(0.0, 0.0);
            fb[m] = m < 8 ? s0[256 + lane + 32 * m] : make_double2(0.0, 0.0);
        }
    }
    __syncwarp();      // the transposes below overwrite the warp's own tile only
    fw::fft512x2<-1>(fa, fb, v, tile, lane, tw512);
    {
        const int line = lane >> 4, k1 = lane & 15;
        __syncwarp();
#pragma unroll
        for (int k2 = 0; k2 < 32; ++k2) tile[line * XSM + k1 + 16 * k2] = v[fw::p32(k2)];
        __syncwarp();
    }
    constexpr int NI = (XSH + 31) / 32;   // 17
    double2 xo[2][NI];
    const double2 w32 = tw1024[32];
    double2 wk = tw1024[lane];
#pragma unroll
    for (int i = 0; i < NI; ++i) {
        if (i % 4 == 0) { if (i) wk = tw1024[lane + 32 * i]; }
        else wk = cmul(wk, w32);
#pragma unroll
        for (int ln = 0; ln < 2; ++ln) {
            const int kx = lane + 32 * i;
            if (kx < XSH) {
                const double2 zk = tile[ln * XSM + (kx & (XSM - 1))];
                const double2 zm = tile[ln * XSM + ((XSM - kx) & (XSM - 1))];
                const double2 Ev = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
                const double2 Od = make_double2(0.5 * (zk.y + zm.y), -0.5 * (zk.x - zm.x));
                xo[ln][i] = cadd(Ev, cmul(wk, Od));
            }
        }
    }
    __syncthreads();   // every warp is done with its tile: stage the slice
#pragma unroll
    for (int ln = 0; ln < 2; ++ln)
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            const int kx = lane + 32 * i;
            if (kx < XSH) S[(kx * 2 + ln) * 3 + c] = xo[ln][i];
        }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        tma_store_2d(&map_main, xo0, 0, S);
        tma_store_2d(&map_main, xo0, 256, S + 256 * 6);
        tma_store_2d(&map_tail, xo0, 512, S + 512 * 6);
        bulk_commit();
        bulk_wait_read();
    }
}

bool xstage_eligible(const StageArgs& a) {
    // opt-in (MXB_XFUSE=1): measured slower than the unfused kernels at 512^3
    // (DESIGN.md section 4); read per call, tests switch it
    const char* e = getenv("MXB_XFUSE");
    if (!e || e[0] != '1') return false;
    const Grid& g = a.g;
    return a.mat.uniform && a.mat.all_magnetic && a.ghost != MXB_GHOST_PERIODIC &&
           !(a.terms & (MXB_TERM_CUBIC | MXB_TERM_BULK_DMI)) && (a.terms & MXB_TERM_DEMAG) &&
           !a.halo_lo && !a.halo_hi && g.nx == XSM && ((long long)g.ny * g.nz) % 2 == 0;
}

template <int MODE, bool E, bool R2C>
static void launch_x1(const StageArgs& a, const XStage& x, const CUtensorMap& mm, const CUtensorMap& mt,
                      unsigned grid, cudaStream_t st) {
    const size_t smem = (size_t)2 * XSH * 3 * sizeof(double2);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_stage_x<MODE, E, R2C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_stage_x<MODE, E, R2C>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        attr = true;
    }
    k_stage_x<MODE, E, R2C><<<grid, 96, smem, st>>>(a, x.tw512, x.tw1024, mm, mt);
}

template <int MODE, bool R2C>
static void launch_x2(bool exact, const StageArgs& a, const XStage& x, const CUtensorMap& mm,
                      const CUtensorMap& mt, unsigned grid, cudaStream_t st) {
    if (exact) launch_x1<MODE, true, R2C>(a, x, mm, mt, grid, st);
    else launch_x1<MODE, false, R2C>(a, x, mm, mt, grid, st);
}

int launch_xstage(int mode, bool exact, const StageArgs& a0, const XStage& x, cudaStream_t st) {
    StageArgs a = a0;
    const long long rows = (long long)a.g.ny * a.g.nz;
    const unsigned grid = (unsigned)(rows / 2);
    // the plane-major slice [kx][row][3] as a 2-D float64 tensor (k_c2r_w's maps)
    CUtensorMap mm{}, mt{};
    const unsigned long long inner = (unsigned long long)rows * 6, pitch_b = (unsigned long long)x.blke * 16;
    int rc;
    if ((rc = make_map_2d_f64(&mm, x.X, inner, XSH, pitch_b, 12, 256)) ||
        (rc = make_map_2d_f64(&mt, x.X, inner, XSH, pitch_b, 12, 1)))
        return rc;
    a.nparts = (int)grid;
    switch (mode) {
        case M_RK1: launch_x2<M_RK1, true>(exact, a, x, mm, mt, grid, st); break;
        case M_RK2: launch_x2<M_RK2, true>(exact, a, x, mm, mt, grid, st); break;
        case M_RK3: launch_x2<M_RK3, true>(exact, a, x, mm, mt, grid, st); break;
        case M_RK4: launch_x2<M_RK4, false>(exact, a, x, mm, mt, grid, st); break;
        default: set_error("x-row fused stage: RK4 stages only"); return MXB_EINVAL;
    }
    MXB_LAUNCH_CHECK();
    if (mode == M_RK4) return launch_finalize(a, 0, st);
    return MXB_OK;
}

}  // namespace mxb
