// Warp-per-line FFT of length 1024 = 32 x 32 (four-step), for the fast path.
//
// A whole line lives in one warp: lane l holds the 32 points x[l + 32 m].
//   1. a 32-point DFT over m in registers (4 x 8 split, constant twiddles)
//   2. twiddle by w1024^(l k) from the exact table
//   3. one transpose through a warp-private 16 KB shared tile (XOR swizzle,
//      bank-conflict free both ways, __syncwarp only)
//   4. a 32-point DFT over l in registers
// Output: lane j holds X[j + 32 k] in register p(k) = 8 (k % 4) + k / 4.
// Compared with the CTA-wide radix-16 Stockham core (fft_fast.cuh) this is
// one shared-memory exchange instead of two and no CTA barrier; zero-padded
// inputs and unneeded outputs fold away at compile time (registers that are
// constant zero / never stored).
#pragma once

#ifndef MXB_HALF_IN
#define MXB_HALF_IN 1   // zero-padded forward inputs skip the zero half of the first stage
#endif
#ifndef MXB_FFT_TW2
#define MXB_FFT_TW2 1   // two interleaved twiddle chains in fft1024: pipeline 80.8 -> 79.3 ms per step
#endif
#ifndef MXB_FFT_TW4
#define MXB_FFT_TW4 1   // four interleaved chains (one per 8-block): another -0.3%, no spills
#endif
#ifndef MXB_FFT512_TW2
#define MXB_FFT512_TW2 1   // fft512x2: chains k and k + 8 interleaved (x passes -0.8%)
#endif

#include "fft_fast.cuh"
#include "fft_generic.cuh"

namespace mxb {
namespace fw {

// a * exp(DIR * 2 pi i e / 32); e is a compile-time constant after unrolling
template <int DIR> __device__ __forceinline__ double2 w32(double2 a, int e) {
    e &= 31;
    if (e == 0) return a;
    if (e == 8) return mul_mi<DIR>(a);
    if (e == 16) return make_double2(-a.x, -a.y);
    if (e == 24) return mul_mi<-DIR>(a);
    double c, s;
    switch (e) {
        case 0: c = 1.000000000000000000000000; s = 0.0; break;
        case 1: c = 0.9807852804032304491261822; s = 0.1950903220161282678482849; break;
        case 2: c = 0.9238795325112867561281832; s = 0.3826834323650897717284600; break;
        case 3: c = 0.8314696123025452370787884; s = 0.5555702330196022247428308; break;
        case 4: c = 0.7071067811865475244008444; s = 0.7071067811865475244008444; break;
        case 5: c = 0.5555702330196022247428308; s = 0.8314696123025452370787884; break;
        case 6: c = 0.3826834323650897717284600; s = 0.9238795325112867561281832; break;
        case 7: c = 0.1950903220161282678482849; s = 0.9807852804032304491261822; break;
        case 8: c = 2.067032109826398823649690e-43; s = 1.000000000000000000000000; break;
        case 9: c = -0.1950903220161282678482849; s = 0.9807852804032304491261822; break;
        case 10: c = -0.3826834323650897717284600; s = 0.9238795325112867561281832; break;
        case 11: c = -0.5555702330196022247428308; s = 0.8314696123025452370787884; break;
        case 12: c = -0.7071067811865475244008444; s = 0.7071067811865475244008444; break;
        case 13: c = -0.8314696123025452370787884; s = 0.5555702330196022247428308; break;
        case 14: c = -0.9238795325112867561281832; s = 0.3826834323650897717284600; break;
        case 15: c = -0.9807852804032304491261822; s = 0.1950903220161282678482849; break;
        case 16: c = -1.000000000000000000000000; s = 4.134064219652797647299381e-43; break;
        case 17: c = -0.9807852804032304491261822; s = -0.1950903220161282678482849; break;
        case 18: c = -0.9238795325112867561281832; s = -0.3826834323650897717284600; break;
        case 19: c = -0.8314696123025452370787884; s = -0.5555702330196022247428308; break;
        case 20: c = -0.7071067811865475244008444; s = -0.7071067811865475244008444; break;
        case 21: c = -0.5555702330196022247428308; s = -0.8314696123025452370787884; break;
        case 22: c = -0.3826834323650897717284600; s = -0.9238795325112867561281832; break;
        case 23: c = -0.1950903220161282678482849; s = -0.9807852804032304491261822; break;
        case 24: c = 2.233876440654988324291948e-41; s = -1.000000000000000000000000; break;
        case 25: c = 0.1950903220161282678482849; s = -0.9807852804032304491261822; break;
        case 26: c = 0.3826834323650897717284600; s = -0.9238795325112867561281832; break;
        case 27: c = 0.5555702330196022247428308; s = -0.8314696123025452370787884; break;
        case 28: c = 0.7071067811865475244008444; s = -0.7071067811865475244008444; break;
        case 29: c = 0.8314696123025452370787884; s = -0.5555702330196022247428308; break;
        case 30: c = 0.9238795325112867561281832; s = -0.3826834323650897717284600; break;
        case 31: c = 0.9807852804032304491261822; s = -0.1950903220161282678482849; break;
        default: c = 1.0; s = 0.0;
    }
    if (DIR < 0) s = -s;
    return make_double2(a.x * c - a.y * s, a.x * s + a.y * c);
}

// in place; v[8 k1 + k2] = X[k1 + 4 k2] on exit (input natural order)
template <int DIR> __device__ __forceinline__ void dft32(double2 (&v)[32]) {
#pragma unroll
    for (int n2 = 0; n2 < 8; ++n2) {
        double2 q[4] = {v[n2], v[8 + n2], v[16 + n2], v[24 + n2]};
        dft4<DIR>(q);
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) v[8 * k1 + n2] = w32<DIR>(q[k1], n2 * k1);
    }
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) dft8<DIR>(&v[8 * k1]);
}

// dft32 for inputs v[16..31] == 0 (a zero-padded line): the first radix-4
// stage reduces to {a + b, a - i b, a - b, a + i b} (DIR = -1 sign shown), and
// the zero registers are never read.  Equal to dft32 up to the sign of zeros
// (x + 0 is not foldable to x under IEEE rules, so the compiler keeps them).
template <int DIR> __device__ __forceinline__ void dft32_half(double2 (&v)[32]) {
#pragma unroll
    for (int n2 = 0; n2 < 8; ++n2) {
        const double2 a = v[n2], b = v[8 + n2];
        const double2 ib = mul_mi<DIR>(b);
        const double2 q[4] = {cadd(a, b), cadd(a, ib), csub(a, b), csub(a, ib)};
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) v[8 * k1 + n2] = w32<DIR>(q[k1], n2 * k1);
    }
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) dft8<DIR>(&v[8 * k1]);
}

__host__ __device__ constexpr int p32(int k) { return 8 * (k % 4) + k / 4; }

// transpose tile: row r (the step-1 frequency), column l (the lane)
__device__ __forceinline__ int tsw(int r, int l) { return r * 32 + (l ^ (r & 7)); }

// v[m] = x[lane + 32 m] on entry; lane j holds X[j + 32 k] in v[p32(k)] on exit.
// W: this warp's 1024-element tile (free on entry, clobbered).
// HALF_IN: x[n] == 0 for n >= 512 (v[16..31] are not read).
template <int DIR, bool HALF_IN = false>
__device__ __forceinline__ void fft1024(double2 (&v)[32], double2* W, int lane_in, const double2* __restrict__ tw) {
    // an opaque copy of the lane index: the lane-dependent tile addresses are
    // then recomputed per call instead of being hoisted out of the caller's
    // loop (32 live addresses that end up spilled)
    int lane = lane_in;
    asm volatile("" : "+r"(lane));
    if (HALF_IN) dft32_half<DIR>(v);
    else dft32<DIR>(v);
    __syncwarp();
    // w1024^(lane k) as a running product, re-anchored from the exact table
    // every 8 steps (<= 7 products; loading all 31 would pin ~120 registers)
    const double2 w1 = twid<DIR>(tw, lane);
#if MXB_FFT_TW4
    // four interleaved running products, one per 8-block of k, each anchored
    // at the exact table value of its first k
    double2 wq[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) wq[j] = j ? twid<DIR>(tw, lane * 8 * j) : make_double2(1.0, 0.0);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (k) wq[j] = (k == 1 && j == 0) ? w1 : cmul(wq[j], w1);
            const int kk = 8 * j + k;
            const double2 a = kk ? cmul(v[p32(kk)], wq[j]) : v[p32(kk)];
            W[tsw(kk, lane)] = a;
            wq[j].x = fma(0.0, a.x, wq[j].x);
        }
    }
#elif MXB_FFT_TW2
    // two interleaved running products (k and k + 16), each re-anchored from the
    // exact table every 8 steps: half the serial twiddle chain
    double2 wa = make_double2(1.0, 0.0), wb = twid<DIR>(tw, lane * 16);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        if (k & 7) {
            wa = k == 1 ? w1 : cmul(wa, w1);
            wb = cmul(wb, w1);
        } else if (k) {
            wa = twid<DIR>(tw, lane * k);
            wb = twid<DIR>(tw, lane * (k + 16));
        }
        const double2 a = k ? cmul(v[p32(k)], wa) : v[p32(k)];
        const double2 b = cmul(v[p32(k + 16)], wb);
        W[tsw(k, lane)] = a;
        W[tsw(k + 16, lane)] = b;
        wa.x = fma(0.0, a.x, wa.x);
        wb.x = fma(0.0, b.x, wb.x);
    }
#else
    double2 w = make_double2(1.0, 0.0);
#pragma unroll
    for (int k = 0; k < 32; ++k) {
        if (k & 7) w = k == 1 ? w1 : cmul(w, w1);
        else if (k) w = twid<DIR>(tw, lane * k);
        const double2 a = k ? cmul(v[p32(k)], w) : v[p32(k)];
        W[tsw(k, lane)] = a;
        // a real data dependency (0 * a is not foldable under IEEE rules) keeps
        // the twiddle chain in step with the stores; computed ahead, all 31
        // twiddles would stay live across the first DFT
        w.x = fma(0.0, a.x, w.x);
    }
#endif
    __syncwarp();
#pragma unroll
    for (int l = 0; l < 32; ++l) v[l] = W[tsw(lane, l)];
    dft32<DIR>(v);
}


// DFT-16 (as ff::DFT<16>) for inputs x[8..15] == 0
template <int DIR> __device__ __forceinline__ void dft16_half(double2 (&x)[16]) {
    double2 y[16];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const double2 a = x[b], c = x[4 + b];
        const double2 ic = mul_mi<DIR>(c);
        const double2 q[4] = {cadd(a, c), cadd(a, ic), csub(a, c), csub(a, ic)};
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) y[4 * b + k1] = ff::wmul<DIR>(q[k1], b * k1);
    }
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
        double2 q[4] = {y[k1], y[4 + k1], y[8 + k1], y[12 + k1]};
        dft4<DIR>(q);
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) x[k1 + 4 * k2] = q[k2];
    }
}

// Two lines of length 512 = 32 x 16 per warp (the x passes: one line per row
// and component).  Lane l holds xa[l + 32 m] in a[m] and xb[l + 32 m] in b[m]
// (m < 16).  DFT-16 over m in registers, w512^(l k1) twiddles, one transpose
// whose 32 tile rows are (line, k1), DFT-32 over l.  On exit lane j holds
// X_line[k1 + 16 k2] in v[p32(k2)] with line = j >> 4, k1 = j & 15.
// HALF_IN: a[8..15] and b[8..15] are zero (not read).
template <int DIR, bool HALF_IN = false>
__device__ __forceinline__ void fft512x2(double2 (&a)[16], double2 (&b)[16], double2 (&v)[32], double2* W,
                                         int lane_in, const double2* __restrict__ tw512) {
    int lane = lane_in;
    asm volatile("" : "+r"(lane));
    if (HALF_IN) {
        dft16_half<DIR>(a);
        dft16_half<DIR>(b);
    } else {
        ff::DFT<16, DIR>::run(a);
        ff::DFT<16, DIR>::run(b);
    }
    __syncwarp();
    const double2 w1 = twid<DIR>(tw512, lane);
#if MXB_FFT512_TW2
    double2 wa = make_double2(1.0, 0.0), wb = twid<DIR>(tw512, lane * 8);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        if (k) {
            wa = k == 1 ? w1 : cmul(wa, w1);
            wb = cmul(wb, w1);
        }
        const double2 x = k ? cmul(a[k], wa) : a[k];
        const double2 y = k ? cmul(b[k], wa) : b[k];
        const double2 x8 = cmul(a[k + 8], wb), y8 = cmul(b[k + 8], wb);
        W[tsw(k, lane)] = x;
        W[tsw(16 + k, lane)] = y;
        W[tsw(k + 8, lane)] = x8;
        W[tsw(24 + k, lane)] = y8;
        wa.x = fma(0.0, y.x, wa.x);
        wb.x = fma(0.0, y8.x, wb.x);
    }
#else
    double2 w = make_double2(1.0, 0.0);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        if (k & 7) w = k == 1 ? w1 : cmul(w, w1);
        else if (k) w = twid<DIR>(tw512, lane * k);
        const double2 x = k ? cmul(a[k], w) : a[k];
        const double2 y = k ? cmul(b[k], w) : b[k];
        W[tsw(k, lane)] = x;
        W[tsw(16 + k, lane)] = y;
        w.x = fma(0.0, y.x, w.x);
    }
#endif
    __syncwarp();
#pragma unroll
    for (int l = 0; l < 32; ++l) v[l] = W[tsw(lane, l)];
    dft32<DIR>(v);
}

}  // namespace fw
}  // namespace mxb
