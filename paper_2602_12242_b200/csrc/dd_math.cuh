// Correctly rounded (with overwhelming probability) atan and asinh for the
// Newell tensor builder (newell.cu), evaluated in double-double arithmetic.
//
// Why: the reference tensor is three nested second differences of the Newell
// antiderivatives, which are ~r^3 at displacement r while the elements are
// ~1/r^3, so a one-ulp change of a single arcsinh/arctan result moves the
// tensor element by up to r^6 ulp (tests/test_tensor_noise_floor.py).  CUDA's
// asinh/atan carry up to 2-3 ulp of error and differ from numpy's results in
// a large fraction of the lattice points; numpy's (SVML on AVX-512 hosts, glibc
// otherwise) are correctly rounded for all but ~0.03% (arcsinh) / ~0.4%
// (arctan) of the lattice arguments, measured with mpmath.  A correctly
// rounded result therefore reproduces the reference's lattice values on all
// but those points.
//
// Method: table reduction to a small argument (atan: c = k/64, atan(x) =
// atan(c) + atan((x - c)/(1 + xc)); log: m = (1 + j/64)(1 + v)), short
// polynomial in double-double (the leading coefficients in double-double, the
// tail in double), one final rounding.  Relative error of the double-double
// result ~1e-31, so the rounded double is the correctly rounded value unless
// the true value lies within ~1e-31 relative of a rounding boundary.
// Host-callable too (tests/test_dd_math.py checks them against mpmath on CPU
// through tools/dd_math_check.cu).
#pragma once

#include <math.h>

#include "dd_tables.inc"

#if defined(__CUDACC__)
#define DD_FN __host__ __device__ __forceinline__
#else
#define DD_FN inline
#endif

namespace ddm {

#if defined(__CUDACC__)
static __device__ __constant__ const double kAtanTab[65][2] = DD_ATAN_TAB;
static __device__ __constant__ const double kLogTab[65][2] = DD_LOG_TAB;
#endif
static const double kAtanTabH[65][2] = DD_ATAN_TAB;
static const double kLogTabH[65][2] = DD_LOG_TAB;
#if defined(__CUDA_ARCH__)
#define DD_TAB(name) name
#else
#define DD_TAB(name) name##H
#endif

struct dd {
    double hi, lo;
};

DD_FN dd quick_two_sum(double a, double b) {   // |a| >= |b|
    const double s = a + b;
    return {s, b - (s - a)};
}

DD_FN dd two_sum(double a, double b) {
    const double s = a + b;
    const double bb = s - a;
    return {s, (a - (s - bb)) + (b - bb)};
}

DD_FN dd two_prod(double a, double b) {
    const double p = a * b;
    return {p, fma(a, b, -p)};
}

DD_FN dd add(dd a, dd b) {
    dd s = two_sum(a.hi, b.hi);
    const dd t = two_sum(a.lo, b.lo);
    s.lo += t.hi;
    s = quick_two_sum(s.hi, s.lo);
    s.lo += t.lo;
    return quick_two_sum(s.hi, s.lo);
}

DD_FN dd neg(dd a) { return {-a.hi, -a.lo}; }
DD_FN dd sub(dd a, dd b) { return add(a, neg(b)); }

DD_FN dd mul(dd a, dd b) {
    dd p = two_prod(a.hi, b.hi);
    p.lo += a.hi * b.lo + a.lo * b.hi;
    return quick_two_sum(p.hi, p.lo);
}

DD_FN dd mul_d(dd a, double b) {
    dd p = two_prod(a.hi, b);
    p.lo += a.lo * b;
    return quick_two_sum(p.hi, p.lo);
}

DD_FN dd div(dd a, dd b) {
    const double q1 = a.hi / b.hi;
    dd r = sub(a, mul_d(b, q1));
    const double q2 = r.hi / b.hi;
    r = sub(r, mul_d(b, q2));
    const double q3 = r.hi / b.hi;
    const dd q = quick_two_sum(q1, q2);
    return add(q, dd{q3, 0.0});
}

DD_FN dd sqrt_dd(dd a) {   // a > 0
    const double s = sqrt(a.hi);
    const dd e = sub(a, two_prod(s, s));
    return add(dd{s, 0.0}, dd{e.hi / (2.0 * s), 0.0});
}

// atan of w in [0, 1] (double-double in and out)
DD_FN dd atan01(dd w) {
    const int k = (int)(w.hi * 64.0 + 0.5);
    const double c = k * (1.0 / 64.0);
    const dd num = sub(w, dd{c, 0.0});
    const dd den = add(dd{1.0, 0.0}, mul_d(w, c));
    const dd u = div(num, den);            // |u| <= 2^-7
    const dd z = mul(u, u);
    // atan(u) = u (1 - z/3 + z^2/5 - z^3/7 + ... - z^7/15 + z^8/17)
    double q = 1.0 / 17.0;
    q = 1.0 / 15.0 - z.hi * q;
    q = 1.0 / 13.0 - z.hi * q;
    q = 1.0 / 11.0 - z.hi * q;
    q = 1.0 / 9.0 - z.hi * q;
    q = 1.0 / 7.0 - z.hi * q;
    const dd c5 = {0.2, -1.1102230246251566e-17};
    const dd c3 = {0.3333333333333333, 1.850371707708594e-17};
    dd p = sub(c5, mul_d(z, q));
    p = sub(c3, mul(z, p));
    p = sub(dd{1.0, 0.0}, mul(z, p));
    const double* t = DD_TAB(kAtanTab)[k];
    return add(dd{t[0], t[1]}, mul(u, p));
}

DD_FN double atan_cr(double x) {
    if (x != x) return x;
    const bool neg_ = x < 0.0;
    const double t = fabs(x);
    dd r;
    if (t == INFINITY) {
        r = {DD_PIO2_HI, DD_PIO2_LO};
    } else if (t > 1.0) {
        r = sub(dd{DD_PIO2_HI, DD_PIO2_LO}, atan01(div(dd{1.0, 0.0}, dd{t, 0.0})));
    } else {
        r = atan01(dd{t, 0.0});
    }
    const double v = r.hi + r.lo;
    return neg_ ? -v : v;
}

// natural log of a double-double y > 0
DD_FN dd log_dd(dd y) {
    int e;
    double m = frexp(y.hi, &e);     // y.hi = m 2^e, m in [0.5, 1)
    m *= 2.0;
    e -= 1;
    const dd ym = {m, ldexp(y.lo, -e)};
    const int j = (int)((ym.hi - 1.0) * 64.0 + 0.5);
    const double c = 1.0 + j * (1.0 / 64.0);
    const dd v = div(sub(ym, dd{c, 0.0}), dd{c, 0.0});     // |v| <= 2^-7
    const dd s = div(v, add(dd{2.0, 0.0}, v));               // log1p(v) = 2 atanh(s)
    const dd z = mul(s, s);
    double q = 1.0 / 17.0;
    q = 1.0 / 15.0 + z.hi * q;
    q = 1.0 / 13.0 + z.hi * q;
    q = 1.0 / 11.0 + z.hi * q;
    q = 1.0 / 9.0 + z.hi * q;
    q = 1.0 / 7.0 + z.hi * q;
    const dd c5 = {0.2, -1.1102230246251566e-17};
    const dd c3 = {0.3333333333333333, 1.850371707708594e-17};
    dd p = add(c5, mul_d(z, q));
    p = add(c3, mul(z, p));
    p = add(dd{1.0, 0.0}, mul(z, p));
    const dd l1 = mul_d(mul(s, p), 2.0);
    const double* t = DD_TAB(kLogTab)[j];
    dd r = add(dd{t[0], t[1]}, l1);
    const dd el = add(two_prod((double)e, DD_LN2_HI), two_prod((double)e, DD_LN2_LO));
    return add(el, r);
}

DD_FN double asinh_cr(double x) {
    if (x != x || x == 0.0 || fabs(x) == INFINITY) return x;
    const bool neg_ = x < 0.0;
    const double t = fabs(x);
    dd r;
    if (t < 0x1p-20) {
        // t (1 - t^2/6 + 3 t^4/40): the next term is ~2^-120 relative
        const dd z = two_prod(t, t);
        const dd c6 = {0.16666666666666666, 9.25185853854297e-18};
        dd p = sub(c6, dd{z.hi * 0.075, 0.0});
        p = sub(dd{1.0, 0.0}, mul(z, p));
        r = mul_d(p, t);
    } else if (t > 0x1p500) {
        r = add(log_dd(dd{t, 0.0}), dd{DD_LN2_HI, DD_LN2_LO});
    } else {
        // log(t + sqrt(1 + t^2))
        const dd q = add(dd{1.0, 0.0}, two_prod(t, t));
        r = log_dd(add(dd{t, 0.0}, sqrt_dd(q)));
    }
    const double v = r.hi + r.lo;
    return neg_ ? -v : v;
}

// x^2.5 for x > 0 (the point-dipole r^5 of demag.py:136), from x^2 sqrt(x) in
// double-double and one rounding
DD_FN double pow25_cr(double x) {
    const dd s = sqrt_dd(dd{x, 0.0});
    const dd r = mul(two_prod(x, x), s);
    return r.hi + r.lo;
}

}  // namespace ddm
