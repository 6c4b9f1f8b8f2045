// Register-resident Stockham FFT for power-of-two lengths (the fast path).
//
// A line of length L is spread over TPL = L/R threads, each holding R complex
// values in registers.  Stage 0 is a radix-R butterfly on the thread's
// inputs x[t + m*TPL]; later stages exchange through shared memory (one
// padded write + read per stage), radix R except a smaller last radix.
// With R = 16 a 1024-point line needs two exchanges.  The final outputs stay
// in registers: register i holds element out_elem(t, i).
//
// Shared layout: COL (lines fastest, used for strided columns) puts element
// e of line b at pad(e)*NL + b; ROW (used for contiguous x rows) at
// b*(L + L/R + 1) + pad(e).  pad(e) = e + e/R keeps every access pattern of the
// stages bank-conflict free for 16-byte elements.
#pragma once

#include "fft_generic.cuh"

#ifndef MXB_TWIDDLE_PRODUCTS
#define MXB_TWIDDLE_PRODUCTS 1
#endif

namespace mxb {
namespace ff {

__host__ __device__ constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v / 2); }

__host__ __device__ constexpr int last_radix(int L, int R) {
    if (L <= R) return L;
    int ns = R, r = R;
    while (ns < L) {
        r = (L / ns >= R) ? R : L / ns;
        ns *= r;
    }
    return r;
}

template <int DIR> __device__ __forceinline__ double2 wmul(double2 a, int e16) {
    // a * exp(DIR * 2 pi i e16 / 16)
    constexpr double C1 = 0.92387953251128675613, S1 = 0.38268343236508977173;
    constexpr double R2 = 0.70710678118654752440;
    double c, s;
    switch (e16 & 15) {
        case 0: return a;
        case 1: c = C1; s = S1; break;
        case 2: c = R2; s = R2; break;
        case 3: c = S1; s = C1; break;
        case 4: return mul_mi<DIR>(a);
        case 6: c = -R2; s = R2; break;
        case 9: c = -C1; s = -S1; break;
        default: {
            const double ang = 2.0 * 3.14159265358979323846 * (e16 & 15) / 16.0;
            c = cos(ang); s = sin(ang);
        }
    }
    if (DIR < 0) s = -s;
    return make_double2(a.x * c - a.y * s, a.x * s + a.y * c);
}

template <int R, int DIR> struct DFT;
template <int DIR> struct DFT<1, DIR> {
    static __device__ __forceinline__ void run(double2*) {}
};
template <int DIR> struct DFT<2, DIR> {
    static __device__ __forceinline__ void run(double2* x) {
        const double2 a = x[0];
        x[0] = cadd(a, x[1]);
        x[1] = csub(a, x[1]);
    }
};
template <int DIR> struct DFT<4, DIR> {
    static __device__ __forceinline__ void run(double2* x) { dft4<DIR>(x); }
};
template <int DIR> struct DFT<8, DIR> {
    static __device__ __forceinline__ void run(double2* x) { dft8<DIR>(x); }
};
template <int DIR> struct DFT<16, DIR> {
    static __device__ __forceinline__ void run(double2* x) {
        double2 y[16];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            double2 q[4] = {x[b], x[4 + b], x[8 + b], x[12 + b]};
            dft4<DIR>(q);
#pragma unroll
            for (int k1 = 0; k1 < 4; ++k1) y[4 * b + k1] = wmul<DIR>(q[k1], b * k1);
        }
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) {
            double2 q[4] = {y[k1], y[4 + k1], y[8 + k1], y[12 + k1]};
            dft4<DIR>(q);
#pragma unroll
            for (int k2 = 0; k2 < 4; ++k2) x[k1 + 4 * k2] = q[k2];
        }
    }
};

template <bool COL, int L, int R, int NL>
__device__ __forceinline__ int sidx(int b, int e) {
    constexpr int LOGR = ilog2(R);
    const int pe = e + (e >> LOGR);
    if (COL) return pe * NL + b;
    return b * (L + L / R + 1) + pe;   // +1: successive lines start in different banks
}

template <int L, int R, int NL>
__host__ __device__ constexpr int smem_elems() { return NL * (L + L / R + 1); }

// cp.async 16-byte global -> shared copy; pred=false zero-fills (src-size 0)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int sz = pred ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// element index held by register i after the final stage
template <int L, int R>
__device__ __forceinline__ int out_elem(int t, int i) {
    constexpr int TPL = L / R;
    constexpr int rl = last_radix(L, R);
    const int q = i / rl, m = i % rl;
    return t + q * TPL + m * (L / rl);
}

template <int L, int R, int NL, bool COL, int DIR, int Ns>
__device__ __forceinline__ void stages(double2 (&v)[R], double2* s, int b, int t,
                                       const double2* __restrict__ tw) {
    if constexpr (Ns < L) {
        constexpr int r = (L / Ns >= R) ? R : L / Ns;
        constexpr int NQ = R / r;
        constexpr int TPL = L / R;
        constexpr int TS = L / (Ns * r);
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const int j = t + q * TPL;
#pragma unroll
            for (int m = 0; m < r; ++m) v[q * r + m] = s[sidx<COL, L, R, NL>(b, j + m * (L / r))];
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const int j = t + q * TPL;
            const int k = j & (Ns - 1);
#if MXB_TWIDDLE_PRODUCTS
            // twiddles w^m: load the powers of two, build the rest with <= 3 products
            double2 w[r];
            w[0] = make_double2(1.0, 0.0);
#pragma unroll
            for (int p = 1; p < r; p <<= 1) w[p] = twid<DIR>(tw, k * p * TS);
#pragma unroll
            for (int m = 3; m < r; ++m)
                if (m & (m - 1)) w[m] = cmul(w[m & (m - 1)], w[m & -m]);
#pragma unroll
            for (int m = 1; m < r; ++m) v[q * r + m] = cmul(v[q * r + m], w[m]);
#else
            // twiddles w^m straight from the table (L1-resident): no fp64 work
#pragma unroll
            for (int m = 1; m < r; ++m) v[q * r + m] = cmul(v[q * r + m], twid<DIR>(tw, k * m * TS));
#endif
            DFT<r, DIR>::run(&v[q * r]);
        }
        if constexpr (Ns * r < L) {
            __syncthreads();
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const int j = t + q * TPL;
                const int k = j & (Ns - 1);
                const int base = (j & ~(Ns - 1)) * r + k;
#pragma unroll
                for (int m = 0; m < r; ++m) s[sidx<COL, L, R, NL>(b, base + m * Ns)] = v[q * r + m];
            }
            __syncthreads();
            stages<L, R, NL, COL, DIR, Ns * r>(v, s, b, t, tw);
        }
    }
}

// v holds x[t + m*TPL] (m < R) on entry; on exit register i holds X[out_elem(t, i)].
// Begins with a barrier so callers may have been reading the shared buffer.
template <int L, int R, int NL, bool COL, int DIR>
__device__ __forceinline__ void fft_core(double2 (&v)[R], double2* s, int b, int t,
                                         const double2* __restrict__ tw) {
    DFT<R, DIR>::run(v);
    if constexpr (L > R) {
        __syncthreads();
#pragma unroll
        for (int m = 0; m < R; ++m) s[sidx<COL, L, R, NL>(b, t * R + m)] = v[m];
        __syncthreads();
        stages<L, R, NL, COL, DIR, R>(v, s, b, t, tw);
    }
}

}  // namespace ff
}  // namespace mxb
