"""Exhaustive check of the in-kernel SDA division (R-11): for integer sums
s in [0, 255 d] and depths d, the fp32 sequence

    r   = RN32(1/d)                    (host, passed to the kernel)
    q0  = RN32(s * r)                  (FMUL)
    rem = RN32(s - q0 * d)             (FFMA: exact product, one rounding)
    q   = RN32(q0 + rem * r)           (FFMA)

must equal the correctly rounded quotient RN32(s / d) bit for bit (the oracle's
value).  Every step is evaluated exactly with integer arithmetic
(Fraction for the rare sums whose fp64 evaluation is inexact).

    python tools/sda_div_check.py [dmax]     (default: every d <= 257 and the config depths)"""
import sys
from fractions import Fraction

import numpy as np


def rn32_exact(x: Fraction) -> np.float32:
    """Correctly rounded fp32 of a rational (ties to even)."""
    f = np.float32(float(x))           # float(x) is RN64; fix up double rounding below
    cand = [np.nextafter(f, np.float32(-np.inf)), f, np.nextafter(f, np.float32(np.inf))]
    best = min(cand, key=lambda c: (abs(Fraction(float(c)) - x), int(np.frombuffer(np.float32(c).tobytes(), np.uint32)[0]) & 1))
    return np.float32(best)


def check(d: int) -> int:
    s = np.arange(0, 255 * d + 1, dtype=np.float64)
    r = np.float32(1.0 / d) if Fraction(float(np.float32(1.0 / d))) == rn32_exact(Fraction(1, d)) else rn32_exact(Fraction(1, d))
    r64 = np.float64(r)
    q0 = (s * r64).astype(np.float32)                       # s*r exact in fp64 (s < 2^20, r 24 bits)
    rem = (s - q0.astype(np.float64) * d).astype(np.float32)  # q0*d exact, difference exact -> one rounding
    t = rem.astype(np.float64) * r64                        # exact (48 bits)
    y = q0.astype(np.float64) + t                           # may be inexact: detect with TwoSum
    bb = y - q0.astype(np.float64)
    err = (q0.astype(np.float64) - (y - bb)) + (t - bb)
    q = y.astype(np.float32)
    bad = np.nonzero(err != 0)[0]
    for i in bad:                                           # exact evaluation of the FFMA
        q[i] = rn32_exact(Fraction(float(q0[i])) + Fraction(float(rem[i])) * Fraction(float(r)))
    ref = np.array([0], np.float32)
    # correctly rounded s/d: fp64 quotient then fp32, fixed up where the fp64 quotient is inexact at a tie
    ref = (s / d).astype(np.float32)
    near = np.nonzero(np.abs((ref.astype(np.float64) * d - s)) > 0)[0]
    mism = np.nonzero(q.view(np.uint32) != ref.view(np.uint32))[0]
    nbad = 0
    for i in mism:                                          # arbitrate exactly
        exact = rn32_exact(Fraction(int(s[i]), d))
        if q[i].view(np.uint32) != exact.view(np.uint32):
            nbad += 1
    return nbad


if __name__ == "__main__":
    depths = list(range(2, 258)) + [300, 1200, 1800, 3600]
    if len(sys.argv) > 1:
        depths = [d for d in depths if d <= int(sys.argv[1])]
    total = 0
    for d in depths:
        n = check(d)
        total += n
        if n:
            print(f"d={d}: {n} mismatches")
    print(f"checked {len(depths)} depths, {sum(255 * d + 1 for d in depths)} sums: {total} mismatches")
    sys.exit(1 if total else 0)
