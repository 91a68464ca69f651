"""Exhaustive error of convert's fp32 atan polynomial over every float t in [0, 1].

    python tools/fast_atan_bound.py [step]   (step > 1: every step-th float, a quick look)

Evaluates p(t) * t exactly as fast_atan2f does (six FFMA2 lanes of an odd
degree-13 polynomial in s = t*t, then one product), emulating each
single-rounding fp32 FMA as an exact float64 product-sum rounded once to
float32 (a*b is exact in float64, so this is the FMA up to a rare double
rounding: at most one extra float32 ulp, 6e-8 rad), and compares with
float64 arctan.  The maximum is the polynomial + evaluation term of the
fast path's error budget (convert.cu); t itself carries the approximate
reciprocal's error, which the budget adds separately.
"""
import sys

import numpy as np

C = np.array([0.006811790633946657, -0.0336042121052742, 0.07962366193532944, -0.1323334127664566,
              0.19807815551757812, -0.3331736922264099, 0.9999961256980896], np.float32)


def fma32(a, b, c):
    return (a.astype(np.float64) * b.astype(np.float64) + c.astype(np.float64)).astype(np.float32)


def poly(t):
    s2 = (t.astype(np.float64) * t).astype(np.float32)  # t*t rounded
    p = np.full_like(t, C[0])
    for k in C[1:]:
        p = fma32(p, s2, np.float32(k))
    return (p.astype(np.float64) * t).astype(np.float32)


def main():
    step = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    top = np.float32(1.0).view(np.uint32)
    worst, at = 0.0, 0.0
    chunk = 1 << 24
    for lo in range(0, int(top) + 1, chunk * step):
        bits = np.arange(lo, min(lo + chunk * step, int(top) + 1), step, dtype=np.uint32)
        t = bits.view(np.float32)
        e = np.abs(poly(t).astype(np.float64) - np.arctan(t.astype(np.float64)))
        i = int(np.argmax(e))
        if e[i] > worst:
            worst, at = float(e[i]), float(t[i])
    print(f"max |fast_atan(t) - atan(t)| over {'all' if step == 1 else 'every %d-th' % step} float t in [0, 1]: "
          f"{worst:.3e} rad at t = {at:.9g}")


if __name__ == "__main__":
    main()
