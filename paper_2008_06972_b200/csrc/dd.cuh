// Double-double helpers for exact bin decisions near bin edges.
//
// The reference bins with glibc atan2/acos (project_kernel,
// /root/reference/pkg/src/stpc/_kernels.py:337, 346); CUDA's are within 2 ulp
// of the true value, glibc's are (nearly always) correctly rounded.  Far from a
// bin edge the two agree on the bin; within 1e-9 of an edge the convert kernel
// refines the angle to ~100 bits with one Newton step in double-double
// arithmetic and rounds it, reproducing the correctly-rounded result the
// reference sees (e.g. its own 45-degree known answer, which sits exactly on
// an edge).  Explicit __fma_rn is used for exact products; -fmad=false only
// disables implicit contraction.
#pragma once
#include <cuda_runtime.h>

namespace stpc {
namespace dd {

struct D2 {
    double hi, lo;
};

__device__ __forceinline__ D2 two_sum(double a, double b)
{
    double s = __dadd_rn(a, b);
    double bb = __dsub_rn(s, a);
    double err = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
    return {s, err};
}

__device__ __forceinline__ D2 quick_two_sum(double a, double b)
{
    double s = __dadd_rn(a, b);
    return {s, __dsub_rn(b, __dsub_rn(s, a))};
}

__device__ __forceinline__ D2 two_prod(double a, double b)
{
    double p = __dmul_rn(a, b);
    return {p, __fma_rn(a, b, -p)};
}

__device__ __forceinline__ D2 add(D2 a, D2 b)
{
    D2 s = two_sum(a.hi, b.hi);
    D2 t = two_sum(a.lo, b.lo);
    s.lo = __dadd_rn(s.lo, t.hi);
    s = quick_two_sum(s.hi, s.lo);
    s.lo = __dadd_rn(s.lo, t.lo);
    return quick_two_sum(s.hi, s.lo);
}

__device__ __forceinline__ D2 neg(D2 a) { return {-a.hi, -a.lo}; }

__device__ __forceinline__ D2 mul(D2 a, D2 b)
{
    D2 p = two_prod(a.hi, b.hi);
    p.lo = __dadd_rn(p.lo, __dadd_rn(__dmul_rn(a.hi, b.lo), __dmul_rn(a.lo, b.hi)));
    return quick_two_sum(p.hi, p.lo);
}

__device__ __forceinline__ D2 mul_d(D2 a, double b)
{
    D2 p = two_prod(a.hi, b);
    p.lo = __dadd_rn(p.lo, __dmul_rn(a.lo, b));
    return quick_two_sum(p.hi, p.lo);
}

__device__ __forceinline__ D2 div_d(D2 a, double b)
{
    double q1 = __ddiv_rn(a.hi, b);
    D2 r = add(a, neg(two_prod(q1, b)));
    double q2 = __ddiv_rn(r.hi, b);
    return quick_two_sum(q1, q2);
}

__device__ __forceinline__ D2 sqrt_dd(D2 a)
{
    if (a.hi <= 0.0) return {0.0, 0.0};
    double x = sqrt(a.hi);
    D2 r = add(a, neg(two_prod(x, x)));
    return quick_two_sum(x, __ddiv_rn(r.hi, __dmul_rn(2.0, x)));
}

// sin and cos of a double-double angle |a| <~ 8, accurate to ~2^-100.
__device__ inline void sincos_dd(D2 a, D2& s, D2& c)
{
    const D2 PIO2 = {1.5707963267948966, 6.123233995736766e-17};
    const double PIO2_3 = -1.4973849048591698e-33;
    double k = rint(__ddiv_rn(a.hi, 1.5707963267948966));
    // t = a - k*pi/2 with a 3-part pi/2
    D2 t = add(a, neg(mul_d(PIO2, k)));
    t = add(t, D2{-__dmul_rn(k, PIO2_3), 0.0});
    D2 t2 = mul(t, t);
    // Taylor series, |t| <= pi/4: 15 terms keep the tail below 2^-110
    D2 sn = t, term = t;
    for (int i = 1; i <= 14; ++i) {
        term = div_d(mul(term, t2), -(double)((2 * i) * (2 * i + 1)));
        sn = add(sn, term);
    }
    D2 cs = {1.0, 0.0};
    term = {1.0, 0.0};
    for (int i = 1; i <= 14; ++i) {
        term = div_d(mul(term, t2), -(double)((2 * i - 1) * (2 * i)));
        cs = add(cs, term);
    }
    int q = ((int)k) & 3;
    if (q == 0) { s = sn; c = cs; }
    else if (q == 1) { s = cs; c = neg(sn); }
    else if (q == 2) { s = neg(sn); c = neg(cs); }
    else { s = neg(cs); c = sn; }
}

// One Newton step on g(a) = Y cos a - X sin a from a0 ~ atan2(Y, X):
// returns the angle to ~2^-100 (hi = correctly rounded double barring a
// ~2^-100 tie).
__device__ inline D2 atan2_refine(D2 Y, D2 X, double a0)
{
    D2 s, c;
    sincos_dd(D2{a0, 0.0}, s, c);
    D2 num = add(mul(Y, c), neg(mul(X, s)));
    D2 den = add(mul(X, c), mul(Y, s));
    double delta = __ddiv_rn(num.hi, den.hi);
    return two_sum(a0, delta);
}

// Correctly rounded atan2(y, x) (np.arctan2 argument order: y first).
__device__ inline double atan2_cr(double y, double x)
{
    double a0 = atan2(y, x);
    if (a0 == 0.0 || !isfinite(a0)) return a0;
    D2 r = atan2_refine(D2{y, 0.0}, D2{x, 0.0}, a0);
    return __dadd_rn(r.hi, r.lo);
}

// Correctly rounded acos(c), |c| <= 1: atan2(sqrt((1-c)(1+c)), c).
__device__ inline double acos_cr(double cz)
{
    double a0 = acos(cz);
    if (cz >= 1.0 || cz <= -1.0) return a0;
    D2 one_m = two_sum(1.0, -cz);
    D2 one_p = two_sum(1.0, cz);
    D2 s = sqrt_dd(mul(one_m, one_p));
    D2 r = atan2_refine(s, D2{cz, 0.0}, a0);
    return __dadd_rn(r.hi, r.lo);
}

}  // namespace dd
}  // namespace stpc
