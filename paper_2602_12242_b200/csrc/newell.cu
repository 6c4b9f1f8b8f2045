// GPU cell-pair demag tensor (DemagKernel.build, demag.py:37-166).
//
// Same algorithm as the reference: the Newell antiderivatives f/g are
// evaluated once on the (2n+1)^3 displacement lattice in units of the
// cell-volume cube root, the 64-corner sum is taken as three second
// differences (z, then y, then x; (hi - 2 mid) + lo each), divided by 4*pi,
// and elements beyond 60 cell diagonals switch to the point-dipole form.
// Arithmetic runs with explicitly rounded intrinsics (no FMA contraction) in
// the reference's operation order, and arcsinh/arctan (and the dipole r^5)
// are correctly rounded (dd_math.cuh): the lattice values are bitwise the
// reference's wherever numpy's own results are correctly rounded (all but
// ~0.4% of the arctan and ~0.03% of the arcsinh arguments); CUDA's
// asinh/atan (2-3 ulp) moved the field by 5e-10..5e-8 at 32^3..128^3.
//
// symmetric=1 evaluates the non-negative displacement octant only and
// mirrors it with the exact parities (XX,YY,ZZ even; XY odd in x,y; XZ odd in
// x,z; YZ odd in y,z), which makes the spectra exactly real.
#include <math.h>

#include "dd_math.cuh"
#include "demag.cuh"

namespace mxb {

#define A_ add<true>
#define S_ sub<true>
#define M_ mul<true>

__device__ double nf(double x, double y, double z) {
    x = fabs(x); y = fabs(y); z = fabs(z);
    const double x2 = M_(x, x), y2 = M_(y, y), z2 = M_(z, z);
    const double r = sqrt(A_(A_(x2, y2), z2));
    const double sxz = sqrt(A_(x2, z2));
    const double sxy = sqrt(A_(x2, y2));
    const double t1 = M_(M_(M_(0.5, y), S_(z2, x2)), ddm::asinh_cr(sxz > 0 ? div_rn(y, sxz) : 0.0));
    const double t2 = M_(M_(M_(0.5, z), S_(y2, x2)), ddm::asinh_cr(sxy > 0 ? div_rn(z, sxy) : 0.0));
    const double xr = M_(x, r);
    const double t3 = M_(M_(M_(-x, y), z), ddm::atan_cr(xr > 0 ? div_rn(M_(y, z), xr) : 0.0));
    const double t4 = div_rn(M_(S_(S_(M_(2.0, x2), y2), z2), r), 6.0);
    return A_(A_(A_(t1, t2), t3), t4);
}

__device__ __forceinline__ double sdiv(double n, double d) { return d != 0.0 ? div_rn(n, d) : 0.0; }

__device__ double ng(double x, double y, double z) {
    z = fabs(z);
    const double x2 = M_(x, x), y2 = M_(y, y), z2 = M_(z, z);
    const double r = sqrt(A_(A_(x2, y2), z2));
    const double sxy = sqrt(A_(x2, y2)), syz = sqrt(A_(y2, z2)), sxz = sqrt(A_(x2, z2));
    const double t1 = M_(M_(M_(x, y), z), ddm::asinh_cr(sdiv(z, sxy)));
    const double t2 = M_(M_(div_rn(y, 6.0), S_(M_(3.0, z2), y2)), ddm::asinh_cr(sdiv(x, syz)));
    const double t3 = M_(M_(div_rn(x, 6.0), S_(M_(3.0, z2), x2)), ddm::asinh_cr(sdiv(y, sxz)));
    const double t4 = M_(-div_rn(M_(z2, z), 6.0), ddm::atan_cr(sdiv(M_(x, y), M_(z, r))));
    const double t5 = M_(-div_rn(M_(z, y2), 2.0), ddm::atan_cr(sdiv(M_(x, z), M_(y, r))));
    const double t6 = M_(-div_rn(M_(z, x2), 2.0), ddm::atan_cr(sdiv(M_(y, z), M_(x, r))));
    const double t7 = div_rn(M_(M_(-x, y), r), 3.0);
    return A_(A_(A_(A_(A_(A_(t1, t2), t3), t4), t5), t6), t7);
}

// lattice index (iz,iy,ix) in (2nz+1)(2ny+1)(2nx+1); coordinate (i - n) * u
__global__ void k_lattice(double* F, int comp, int nx, int ny, int nz, double ux, double uy,
                          double uz) {
    const long long lx = 2 * nx + 1, ly = 2 * ny + 1, lz = 2 * nz + 1;
    const long long tot = lx * ly * lz;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot;
         t += (long long)gridDim.x * blockDim.x) {
        const long long ix = t % lx, r = t / lx, iy = r % ly, iz = r / ly;
        const double X = M_((double)(ix - nx), ux);
        const double Y = M_((double)(iy - ny), uy);
        const double Z = M_((double)(iz - nz), uz);
        double v;
        switch (comp) {
            case 0: v = nf(X, Y, Z); break;
            case 1: v = ng(X, Y, Z); break;
            case 2: v = ng(X, Z, Y); break;
            case 3: v = nf(Y, Z, X); break;
            case 4: v = ng(Y, Z, X); break;
            default: v = nf(Z, X, Y); break;
        }
        F[t] = v;
    }
}

__device__ __forceinline__ double d2(double lo, double mid, double hi) {
    return A_(S_(hi, M_(2.0, mid)), lo);
}

// tensor element of displacement (dx,dy,dz) (|d| <= n-1) from the lattice
__device__ double element(const double* F, int comp, int nx, int ny, int nz, int dx, int dy,
                          int dz, double ux, double uy, double uz, double far2) {
    const double X = M_((double)dx, ux), Y = M_((double)dy, uy), Z = M_((double)dz, uz);
    const double r2 = A_(A_(M_(X, X), M_(Y, Y)), M_(Z, Z));
    const double c = div_rn(1.0, M_(4.0, 3.141592653589793));
    if (r2 > far2) {
        const double r5 = ddm::pow25_cr(r2);
        switch (comp) {
            case 0: return div_rn(M_(c, S_(M_(M_(3.0, X), X), r2)), r5);
            case 3: return div_rn(M_(c, S_(M_(M_(3.0, Y), Y), r2)), r5);
            case 5: return div_rn(M_(c, S_(M_(M_(3.0, Z), Z), r2)), r5);
            case 1: return div_rn(M_(M_(M_(c, 3.0), X), Y), r5);
            case 2: return div_rn(M_(M_(M_(c, 3.0), X), Z), r5);
            default: return div_rn(M_(M_(M_(c, 3.0), Y), Z), r5);
        }
    }
    const long long lx = 2 * nx + 1, ly = 2 * ny + 1;
    const long long bx = dx + nx - 1, by = dy + ny - 1, bz = dz + nz - 1;
    double fy[3][3];  // after the z difference, indexed [y][x]
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            const long long base = (by + a) * lx + (bx + b);
            fy[a][b] = d2(F[(bz + 0) * lx * ly + base], F[(bz + 1) * lx * ly + base],
                          F[(bz + 2) * lx * ly + base]);
        }
    double fx[3];
#pragma unroll
    for (int b = 0; b < 3; ++b) fx[b] = d2(fy[0][b], fy[1][b], fy[2][b]);
    return div_rn(d2(fx[0], fx[1], fx[2]), M_(4.0, 3.141592653589793));
}

// parity of a component under reflection of each axis: +1 even, -1 odd
__device__ __forceinline__ int parity(int comp, int axis) {
    // comp: 0 XX, 1 XY, 2 XZ, 3 YY, 4 YZ, 5 ZZ; axis 0 x, 1 y, 2 z
    switch (comp) {
        case 1: return axis == 2 ? 1 : -1;
        case 2: return axis == 1 ? 1 : -1;
        case 4: return axis == 0 ? 1 : -1;
        default: return 1;
    }
}

struct NewellArgs {
    int nx, ny, nz, px, py, pz, comp, symmetric;
    double ux, uy, uz, far2;
};

// packed wrap-around layout (demag.py:158-166): index i holds displacement
// d = i (i < n) or i - p (i > p - n); the Nyquist slot stays 0.
__global__ void k_pack(const double* F, double* out, NewellArgs a) {
    const long long tot = (long long)a.px * a.py * a.pz;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot;
         t += (long long)gridDim.x * blockDim.x) {
        const int ix = (int)(t % a.px);
        const long long r = t / a.px;
        const int iy = (int)(r % a.py), iz = (int)(r / a.py);
        int dx = ix < a.nx ? ix : ix - a.px;
        int dy = iy < a.ny ? iy : iy - a.py;
        int dz = iz < a.nz ? iz : iz - a.pz;
        double v = 0.0;
        if (dx > -a.nx && dx < a.nx && dy > -a.ny && dy < a.ny && dz > -a.nz && dz < a.nz) {
            if (a.symmetric) {
                int s = 1;
                if (dx < 0) { s *= parity(a.comp, 0); dx = -dx; }
                if (dy < 0) { s *= parity(a.comp, 1); dy = -dy; }
                if (dz < 0) { s *= parity(a.comp, 2); dz = -dz; }
                v = element(F, a.comp, a.nx, a.ny, a.nz, dx, dy, dz, a.ux, a.uy, a.uz, a.far2);
                if (s < 0) v = -v;
            } else {
                v = element(F, a.comp, a.nx, a.ny, a.nz, dx, dy, dz, a.ux, a.uy, a.uz, a.far2);
            }
        }
        out[t] = v;
    }
}

// tensor_elements layout (6, 2nz-1, 2ny-1, 2nx-1) for one component
__global__ void k_elements(const double* F, double* out, NewellArgs a) {
    const long long ex = 2 * a.nx - 1, ey = 2 * a.ny - 1, ez = 2 * a.nz - 1;
    const long long tot = ex * ey * ez;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot;
         t += (long long)gridDim.x * blockDim.x) {
        const int ix = (int)(t % ex);
        const long long r = t / ex;
        const int iy = (int)(r % ey), iz = (int)(r / ey);
        out[t] = element(F, a.comp, a.nx, a.ny, a.nz, ix - (a.nx - 1), iy - (a.ny - 1),
                         iz - (a.nz - 1), a.ux, a.uy, a.uz, a.far2);
    }
}

static void units(const Grid& g, NewellArgs& a) {
    // s = (dx*dy*dz)^(1/3) (demag.py:97-98), on the host with libm pow
    const double s = pow(g.dx * g.dy * g.dz, 1.0 / 3.0);
    a.ux = g.dx / s; a.uy = g.dy / s; a.uz = g.dz / s;
    const double diag = sqrt(a.ux * a.ux + a.uy * a.uy + a.uz * a.uz);
    const double f = 60.0 * diag;
    a.far2 = f * f;
    a.nx = g.nx; a.ny = g.ny; a.nz = g.nz;
    a.px = g.nx > 1 ? 2 * g.nx : 1;
    a.py = g.ny > 1 ? 2 * g.ny : 1;
    a.pz = g.nz > 1 ? 2 * g.nz : 1;
}

int newell_packed_component(const Grid& g, int comp, int symmetric, double* packed_c,
                            double* lattice, cudaStream_t st) {
    NewellArgs a{};
    units(g, a);
    a.comp = comp;
    a.symmetric = symmetric;
    k_lattice<<<148 * 8, 256, 0, st>>>(lattice, comp, g.nx, g.ny, g.nz, a.ux, a.uy, a.uz);
    MXB_LAUNCH_CHECK();
    k_pack<<<148 * 8, 256, 0, st>>>(lattice, packed_c, a);
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

int newell_elements(const Grid& g, double* out6, double* lattice, cudaStream_t st) {
    NewellArgs a{};
    units(g, a);
    const long long per = (long long)(2 * g.nx - 1) * (2 * g.ny - 1) * (2 * g.nz - 1);
    for (int c = 0; c < 6; ++c) {
        a.comp = c;
        k_lattice<<<148 * 8, 256, 0, st>>>(lattice, c, g.nx, g.ny, g.nz, a.ux, a.uy, a.uz);
        MXB_LAUNCH_CHECK();
        k_elements<<<148 * 8, 256, 0, st>>>(lattice, out6 + c * per, a);
        MXB_LAUNCH_CHECK();
    }
    return MXB_OK;
}

// O(N^2) direct sum over source cells (demag_field_direct, demag.py:225-248):
// one thread per target cell, sources in the reference's order (qz, qy, qx),
// zero-magnetisation sources skipped, each source's contribution formed as
// (N_a0 m0 + N_a1 m1) + N_a2 m2 and accumulated with explicit rounding, so
// the sum is the reference's operation for operation.  n6 in the
// tensor_elements layout (6, 2nz-1, 2ny-1, 2nx-1).
__global__ void k_direct_sum(const double* __restrict__ n6, const double* __restrict__ m,
                             double* __restrict__ h, int nx, int ny, int nz) {
    const long long N = (long long)nx * ny * nz;
    const long long ex = 2 * nx - 1, ey = 2 * ny - 1, per = ex * ey * (2 * nz - 1);
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= N) return;
    const int px = (int)(t % nx), py = (int)((t / nx) % ny), pz = (int)(t / ((long long)nx * ny));
    const int mix[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};
    double acc[3] = {0.0, 0.0, 0.0};
    for (int qz = 0; qz < nz; ++qz)
        for (int qy = 0; qy < ny; ++qy)
            for (int qx = 0; qx < nx; ++qx) {
                const long long q = ((long long)qz * ny + qy) * nx + qx;
                const double m0 = m[q], m1 = m[N + q], m2 = m[2 * N + q];
                if (m0 == 0.0 && m1 == 0.0 && m2 == 0.0) continue;
                const long long e = ((long long)(nz - 1 - qz + pz) * ey + (ny - 1 - qy + py)) * ex +
                                    (nx - 1 - qx + px);
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    const double v = A_(A_(M_(n6[mix[a][0] * per + e], m0), M_(n6[mix[a][1] * per + e], m1)),
                                        M_(n6[mix[a][2] * per + e], m2));
                    acc[a] = A_(acc[a], v);
                }
            }
    h[t] = acc[0];
    h[N + t] = acc[1];
    h[2 * N + t] = acc[2];
}

int direct_sum(const Grid& g, const double* n6, const double* m, double* h, cudaStream_t st) {
    const long long N = g.N;
    k_direct_sum<<<(unsigned)((N + 127) / 128), 128, 0, st>>>(n6, m, h, g.nx, g.ny, g.nz);
    MXB_LAUNCH_CHECK();
    return MXB_OK;
}

}  // namespace mxb
