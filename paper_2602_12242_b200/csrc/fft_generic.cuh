// Generic mixed-radix Stockham FFT on lines held in shared memory.
//
// Any length L is supported: radices 8/4/2 are hand-written butterflies, any
// other factor p (3, 5, 7, 11, ...) runs as a direct p-point DFT.  Twiddles
// come from one table tw[n] = exp(-2*pi*i*n/L).  Line b, element e lives at
// s[b*(L+1) + e] (the +1 pad makes the line-strided butterfly accesses
// bank-conflict free for 16-byte complex values).
#pragma once

#include "common.cuh"

namespace mxb {

struct Plan1D {
    int L;
    int nst;
    int radix[24];
    const double2* tw;
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
// multiply by -i (DIR<0) or +i (DIR>0)
template <int DIR> __device__ __forceinline__ double2 mul_mi(double2 a) {
    return DIR < 0 ? make_double2(a.y, -a.x) : make_double2(-a.y, a.x);
}
template <int DIR> __device__ __forceinline__ double2 twid(const double2* tw, int idx) {
    double2 w = tw[idx];
    if (DIR > 0) w.y = -w.y;
    return w;
}

template <int DIR> __device__ __forceinline__ void bfly2(double2& a, double2& b) {
    double2 t = a;
    a = cadd(t, b);
    b = csub(t, b);
}

template <int DIR> __device__ __forceinline__ void dft4(double2* x) {
    double2 t0 = cadd(x[0], x[2]), t1 = csub(x[0], x[2]);
    double2 t2 = cadd(x[1], x[3]), t3 = mul_mi<DIR>(csub(x[1], x[3]));
    x[0] = cadd(t0, t2);
    x[2] = csub(t0, t2);
    x[1] = cadd(t1, t3);
    x[3] = csub(t1, t3);
}

template <int DIR> __device__ __forceinline__ void dft8(double2* x) {
    const double r = 0.70710678118654752440;
    double2 e[4] = {x[0], x[2], x[4], x[6]};
    double2 o[4] = {x[1], x[3], x[5], x[7]};
    dft4<DIR>(e);
    dft4<DIR>(o);
    // o[k] *= exp(DIR*2*pi*i*k/8)
    double2 w1 = make_double2(r, DIR < 0 ? -r : r);
    double2 w3 = make_double2(-r, DIR < 0 ? -r : r);
    o[1] = cmul(o[1], w1);
    o[2] = mul_mi<DIR>(o[2]);
    o[3] = cmul(o[3], w3);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        x[k] = cadd(e[k], o[k]);
        x[k + 4] = csub(e[k], o[k]);
    }
}

// One Stockham stage: a -> b.  Returns nothing; caller swaps.
template <int DIR>
__device__ void stage_generic(const double2* __restrict__ a, double2* __restrict__ b, int NL,
                              int ld, const Plan1D& p, int r, int Ns, int tid, int nthr) {
    const int L = p.L;
    const int nb = L / r;
    const int total = nb * NL;
    const int tstep = L / (Ns * r);
    if (r == 2 || r == 4 || r == 8) {
        for (int u = tid; u < total; u += nthr) {
            const int line = u % NL, j = u / NL, k = j % Ns;
            const double2* src = a + line * ld + j;
            double2 x[8];
#pragma unroll
            for (int m = 0; m < 8; ++m)
                if (m < r) x[m] = src[m * nb];
            if (Ns > 1) {
#pragma unroll
                for (int m = 1; m < 8; ++m)
                    if (m < r) x[m] = cmul(x[m], twid<DIR>(p.tw, k * m * tstep));
            }
            if (r == 2) bfly2<DIR>(x[0], x[1]);
            else if (r == 4) dft4<DIR>(x);
            else dft8<DIR>(x);
            double2* dst = b + line * ld + (j / Ns) * Ns * r + k;
#pragma unroll
            for (int m = 0; m < 8; ++m)
                if (m < r) dst[m * Ns] = x[m];
        }
    } else {
        // direct r-point DFT; one thread per output q of one butterfly
        const int tot2 = total * r;
        const int rstep = L / r;
        for (int u = tid; u < tot2; u += nthr) {
            const int line = u % NL;
            const int rest = u / NL;
            const int q = rest % r, j = rest / r, k = j % Ns;
            const double2* src = a + line * ld + j;
            double2 acc = make_double2(0.0, 0.0);
            for (int m = 0; m < r; ++m) {
                double2 v = src[m * nb];
                if (Ns > 1 && m > 0) v = cmul(v, twid<DIR>(p.tw, k * m * tstep));
                const int qm = (q * m) % r;
                v = qm ? cmul(v, twid<DIR>(p.tw, qm * rstep)) : v;
                acc = cadd(acc, v);
            }
            b[line * ld + (j / Ns) * Ns * r + k + q * Ns] = acc;
        }
    }
}

// Full transform of NL lines; data starts in `a`, result pointer returned.
template <int DIR>
__device__ double2* fft_lines(double2* a, double2* b, int NL, const Plan1D& p, int tid,
                              int nthr) {
    const int ld = p.L + 1;
    int Ns = 1;
    for (int s = 0; s < p.nst; ++s) {
        const int r = p.radix[s];
        stage_generic<DIR>(a, b, NL, ld, p, r, Ns, tid, nthr);
        __syncthreads();
        double2* t = a;
        a = b;
        b = t;
        Ns *= r;
    }
    return a;
}

}  // namespace mxb
