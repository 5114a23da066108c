"""Lifting factorisation of the 8-tap Daubechies analysis pair (R-27).

The analysis a[k] = sum_i H_[i] x[2k-6+i], d[k] = sum_i G_[i] x[2k-6+i] (R-5 in the
GPU's index convention, G_[i] = (-1)^i H_[7-i]) is written in polyphase form
(e[m] = x[2m], o[m] = x[2m+1]) as a 2x2 matrix of Laurent polynomials and
reduced to the identity by lifting steps (the Euclidean algorithm of
Daubechies & Sweldens, 1998), removing the LEADING coefficient at each step
(the ordering whose coefficients stay small: max 1.69; removing the trailing one
gives a step of 16.3).  Prints the constants analysis.cu uses (LF_*) and checks
(1) the cascade reproduces the direct filter in fp64 and (2) its fp32 error.

    python tools/lifting.py"""
import numpy as np

# R-2's filter in the GPU's order (common.cuh PRNU_H0..7)
H = np.array([0.2303778133088965, 0.7148465705529157, 0.6308807679298589, -0.027983769416859854,
              -0.18703481171909309, 0.030841381835560764, 0.0328830116668852, -0.010597401785069032])
G = np.array([(-1) ** i * H[7 - i] for i in range(8)])


# Laurent polynomial: (lowest power, coefficients); the power s acts as v[k] -> v[k + s]
def trim(p, tol=1e-13):
    lo, c = p
    nz = np.nonzero(np.abs(c) > tol)[0]
    return (0, np.zeros(0)) if len(nz) == 0 else (lo + nz[0], c[nz[0]:nz[-1] + 1].copy())


def add(p, q):
    if len(p[1]) == 0:
        return q
    if len(q[1]) == 0:
        return p
    lo = min(p[0], q[0])
    hi = max(p[0] + len(p[1]), q[0] + len(q[1]))
    c = np.zeros(hi - lo)
    c[p[0] - lo:p[0] - lo + len(p[1])] += p[1]
    c[q[0] - lo:q[0] - lo + len(q[1])] += q[1]
    return trim((lo, c))


def mul(p, q):
    if len(p[1]) == 0 or len(q[1]) == 0:
        return (0, np.zeros(0))
    return trim((p[0] + q[0], np.convolve(p[1], q[1])))


def neg(p):
    return (p[0], -p[1])


def quotient(A, B, nterms):
    """q with nterms terms cancelling A's leading coefficient (1 term) or both ends (2)."""
    la, lb = len(A[1]), len(B[1])
    s_hi = A[0] + la - 1 - (B[0] + lb - 1)
    q = (s_hi, np.array([A[1][-1] / B[1][-1]]))
    if nterms == 2:
        q = add((A[0] - B[0], np.array([A[1][0] / B[1][0]])), q)
    return q


def factor():
    # a = He e + Ho o, d = Ge e + Go o with x[2k-6+i]: i even -> e[k-3+i/2], i odd -> o[k-3+(i-1)/2]
    poly = lambda c, par: trim((-3, np.array([c[2 * p + par] for p in range(4)])))
    M = [[poly(H, 0), poly(H, 1)], [poly(G, 0), poly(G, 1)]]
    steps = []

    def colop(i, j, q):   # column j += column i * q  <=>  input component i -= q(S) * component j
        for r in range(2):
            M[r][j] = add(M[r][j], mul(M[r][i], q))
        steps.append((i, j, q))

    colop(0, 1, neg(quotient(M[0][1], M[0][0], 1)))
    while len(M[0][0][1]) and len(M[0][1][1]):
        i, j = (1, 0) if len(M[0][0][1]) >= len(M[0][1][1]) else (0, 1)
        A, B = M[0][j], M[0][i]
        colop(i, j, neg(quotient(A, B, 2 if len(A[1]) == len(B[1]) + 1 else 1)))
    return M, steps


def main():
    M, steps = factor()
    assert [len(s[2][1]) for s in steps] == [1, 2, 2, 2]
    (q1, q2, q3, q4) = [s[2] for s in steps]
    C1 = q1[1][0]
    C2A, C2B = -q2[1][0], q2[1][1]
    C3A, C3B = -q3[1][0], q3[1][1]
    C4A, C4B = -q4[1][0], -q4[1][1]
    KA = M[0][1][1][0]
    KD, c3 = M[1][0][1][0], M[1][1][1][0]
    C5 = -c3 / KD
    for name, v in (("LF_C1", C1), ("LF_C2A", C2A), ("LF_C2B", C2B), ("LF_C3A", C3A), ("LF_C3B", C3B),
                    ("LF_C4A", C4A), ("LF_C4B", C4B), ("LF_C5", C5), ("LF_KA", KA), ("LF_KD", KD),
                    ("LF_KA2", KA * KA), ("LF_KD2", KD * KD), ("LF_KD4", KD ** 4)):
        print(f"#define {name} {float(v)!r}f")
    print("KA*KD - 1 =", KA * KD - 1.0)
    rng = np.random.default_rng(0)
    x = rng.uniform(0, 255, 200)
    err = max(np.abs(lift(x, C1, C2A, C2B, C3A, C3B, C4A, C4B, C5, KA, KD, np.float64) - direct(x, np.float64)).max()
              for _ in range(1))
    print("fp64 lifting vs direct:", err)
    e32l = e32d = 0.0
    for _ in range(50):
        x = rng.integers(0, 256, 200).astype(np.float64)
        ref = direct(x, np.float64)
        e32l = max(e32l, np.abs(lift(x, C1, C2A, C2B, C3A, C3B, C4A, C4B, C5, KA, KD, np.float32) - ref).max())
        e32d = max(e32d, np.abs(direct(x, np.float32) - ref).max())
    print(f"fp32 max error on u8 data: lifting {e32l:.3g}, direct {e32d:.3g}")


def direct(x, dt):
    x = x.astype(dt)
    n = len(x) // 2
    out = np.zeros((2, n - 6))
    for k in range(3, n - 3):
        a = d = dt(0)
        for i in range(8):
            a = dt(a + dt(H[i]) * x[2 * k - 6 + i])
            d = dt(d + dt(G[i]) * x[2 * k - 6 + i])
        out[:, k - 3] = (a, d)
    return out


def lift(x, C1, C2A, C2B, C3A, C3B, C4A, C4B, C5, KA, KD, dt):
    """The cascade in the order analysis.cu evaluates it (numpy rounds each product and sum
    separately; the kernel's FFMA2 rounds once per multiply-add)."""
    c = [dt(v) for v in (C1, C2A, C2B, C3A, C3B, C4A, C4B, C5, KA, KD)]
    C1, C2A, C2B, C3A, C3B, C4A, C4B, C5, KA, KD = c
    x = x.astype(dt)
    e, o = x[0::2], x[1::2]
    n = len(e)
    e1 = e - C1 * o
    o1 = np.zeros(n, dt)
    e2 = np.zeros(n, dt)
    o2 = np.zeros(n, dt)
    e3 = np.zeros(n, dt)
    o1[:-1] = o[:-1] + C2A * e1[:-1] - C2B * e1[1:]
    e2[1:] = e1[1:] + C3A * o1[:-1] - C3B * o1[1:]
    o2[:-1] = o1[:-1] + C4A * e2[:-1] + C4B * e2[1:]
    e3[1:] = e2[1:] - C5 * o2[:-1]
    out = np.zeros((2, n - 6))
    for k in range(3, n - 3):
        out[:, k - 3] = (KA * o2[k - 2], KD * e3[k - 1])
    return out


if __name__ == "__main__":
    main()
