"""f3 denoiser variants (readings R-24..R-26 of DESIGN.md), fp64 numpy.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): never imported by the product
path, and it imports nothing from it.

S:117 names the denoiser "Daubechies-8 ... undecimated-boundary-safe" (garbled)
and S:150 "symmetric (mirror)"; SURVEY Q2-Q4 read the default as the decimated
8-tap transform with half-sample symmetric extension (oracle.c) and list three
alternatives, built here step by step:

* taps = 16  (Q2): db8, the 16-tap Daubechies filter with 8 vanishing moments,
  from the spectral factorisation of the Daubechies polynomial (`daubechies`).
* boundary = 1  (Q4, R-24): pad the plane to a multiple of 2^levels with the
  half-sample symmetric map e_N (bottom / right), periodic (circular) decimated
  DWT, the same shrink, inverse, crop back to H x W.
* transform = 1  (Q3, R-25): undecimated (stationary) DWT: level l filters the
  previous approximation with the filters dilated by s = 2^(l-1), no
  decimation, circular indexing; synthesis is the adjoint / 2 per dimension.

The shrink is the same for every variant: oracle.c's fp64 local-variance Wiener
rule with mirror-extended windows (R-7), applied to every detail subband.  The
residual is W = I - F(I).
"""
from __future__ import annotations

import numpy as np
from math import comb

from . import shrink as _shrink, zero_mean as _zero_mean, DEFAULT_SIGMA0_SQ, DEFAULT_WINDOWS, DEFAULT_LEVELS


# ------------------------------------------------------------------ filters
def daubechies(p: int) -> np.ndarray:
    """dec_lo of the Daubechies wavelet with p vanishing moments (2p taps), fp64.

    Daubechies' construction: H(z) = sqrt(2) ((1 + z^-1)/2)^p Q(z) with
    |Q(e^{iw})|^2 = P(sin^2(w/2)), P(y) = sum_{k<p} C(p-1+k, k) y^k.  Each root
    y_i of P gives the pair (z, 1/z) of roots of z + 1/z = 2 - 4 y_i (since
    y = sin^2(w/2) = (2 - z - 1/z)/4); Q keeps the one inside the unit circle
    (minimum phase).  The result is normalised to sum sqrt(2), and reversed into
    the dec_lo orientation of oracle.c (for p = 4 this reproduces its DEC_LO).
    Rooting P in y (degree p-1) and mapping each root is far better conditioned
    than rooting the degree-2p-2 polynomial in z.
    """
    Py = [float(comb(p - 1 + k, k)) for k in range(p)][::-1]   # highest power first
    zs = []
    for y in np.roots(Py):
        pair = np.roots([1.0, -(2.0 - 4.0 * y), 1.0])          # z^2 - (2 - 4y) z + 1 = 0
        zs.append(pair[np.argmin(np.abs(pair))])
    assert len(zs) == p - 1
    h = np.real(np.poly(zs))                        # Q(z) up to scale (roots in conjugate pairs)
    for _ in range(p):
        h = np.convolve(h, [1.0, 1.0])              # (1 + z^-1)^p
    h = h * (np.sqrt(2.0) / h.sum())
    # np.poly gives the coefficients of z^(n) ... z^0, i.e. the minimum-phase
    # impulse response h[0..2p-1] in increasing delay; dec_lo is its reverse
    return h[::-1].copy()


def qmf(dec_lo: np.ndarray):
    """(dec_lo, dec_hi, rec_lo, rec_hi) by the quadrature-mirror relations of oracle.c:
    dec_hi[k] = (-1)^(k+1) dec_lo[L-1-k]; rec_lo[k] = dec_lo[L-1-k]; rec_hi[k] = dec_hi[L-1-k]."""
    L = len(dec_lo)
    k = np.arange(L)
    dec_hi = np.where(k % 2 == 1, 1.0, -1.0) * dec_lo[::-1]
    return dec_lo, dec_hi, dec_lo[::-1].copy(), dec_hi[::-1].copy()


def filters_for(taps: int):
    if taps == 8:
        return qmf(daubechies(4))
    if taps == 16:
        return qmf(daubechies(8))
    raise ValueError("taps must be 8 or 16")


# ------------------------------------------------------------------ index maps
def ext_sym(i, N: int):
    """e_N (R-4): half-sample symmetric, period 2N."""
    r = np.mod(i, 2 * N)
    return np.where(r < N, r, 2 * N - 1 - r)


def ext_pad_per(i, N: int, Np: int):
    """Periodic with period Np over a plane padded from N to Np by e_N (R-24)."""
    r = np.mod(i, Np)
    return ext_sym(r, N)


# ------------------------------------------------------------------ 1-D transforms (along axis 0)
def dwt_sym(x, lo, hi):
    """Expansive symmetric analysis (R-5 with L taps): n = floor((N + L - 1)/2),
    a[k] = sum_j lo[j] x[e_N(2k+1-j)], d likewise with hi."""
    N, L = x.shape[0], len(lo)
    n = (N + L - 1) // 2
    k = np.arange(n)
    a = np.zeros((n,) + x.shape[1:])
    d = np.zeros((n,) + x.shape[1:])
    for j in range(L):
        v = x[ext_sym(2 * k + 1 - j, N)]
        a += lo[j] * v
        d += hi[j] * v
    return a, d


def idwt_sym(a, d, rl, rh, N: int):
    """Expansive symmetric synthesis: x[t] = sum_k a[k] rl[t+L-2-2k] + d[k] rh[t+L-2-2k],
    terms whose filter index lies in [0, L) (oracle.c's offset 6 for L = 8).  Summed
    per filter index f: coefficient k lands on t = 2k + f - (L-2), kept when 0 <= t < N."""
    n, L = a.shape[0], len(rl)
    x = np.zeros((N,) + a.shape[1:])
    k = np.arange(n)
    for f in range(L):
        t = 2 * k + f - (L - 2)
        ok = (t >= 0) & (t < N)
        x[t[ok]] += a[ok] * rl[f] + d[ok] * rh[f]
    return x


def dwt_per(x, lo, hi, N: int | None = None, Np: int | None = None):
    """Periodic decimated analysis (R-24): a[k] = sum_j lo[j] x[(2k+1-j) mod Np], k < Np/2.
    With N < Np the samples beyond N are the e_N mirror padding."""
    if N is None:
        N = x.shape[0]
    if Np is None:
        Np = N
    assert Np % 2 == 0
    n = Np // 2
    k = np.arange(n)
    a = np.zeros((n,) + x.shape[1:])
    d = np.zeros((n,) + x.shape[1:])
    for j in range(len(lo)):
        v = x[ext_pad_per(2 * k + 1 - j, N, Np)]
        a += lo[j] * v
        d += hi[j] * v
    return a, d


def idwt_per(a, d, lo, hi):
    """Periodic decimated synthesis = the transpose of dwt_per (the transform is
    orthogonal): x[(2k+1-j) mod Np] += lo[j] a[k] + hi[j] d[k]."""
    n = a.shape[0]
    Np = 2 * n
    x = np.zeros((Np,) + a.shape[1:])
    k = np.arange(n)
    for j in range(len(lo)):
        np.add.at(x, np.mod(2 * k + 1 - j, Np), lo[j] * a + hi[j] * d)
    return x


def dwt_swt(x, lo, hi, s: int):
    """Undecimated analysis at dilation s (R-25): a[t] = sum_j lo[j] x[(t - s j) mod N]."""
    N = x.shape[0]
    t = np.arange(N)
    a = np.zeros_like(x, dtype=np.float64)
    d = np.zeros_like(x, dtype=np.float64)
    for j in range(len(lo)):
        v = x[np.mod(t - s * j, N)]
        a += lo[j] * v
        d += hi[j] * v
    return a, d


def idwt_swt(a, d, lo, hi, s: int):
    """Undecimated synthesis: half the adjoint, x[t] = 1/2 sum_j lo[j] a[(t + s j) mod N] + hi[j] d[...]
    (the analysis pair is a tight frame with bound 2: |H|^2 + |G|^2 = 2)."""
    N = a.shape[0]
    t = np.arange(N)
    x = np.zeros_like(a, dtype=np.float64)
    for j in range(len(lo)):
        idx = np.mod(t + s * j, N)
        x += lo[j] * a[idx] + hi[j] * d[idx]
    return 0.5 * x


# ------------------------------------------------------------------ 2-D levels (rows, then columns; R-6)
def _along_x(f, *planes_and_args, n_planes: int = 1):
    """Apply a 1-D axis-0 transform along x (the last axis) of 2-D planes."""
    planes = [np.swapaxes(p, 0, 1) for p in planes_and_args[:n_planes]]
    out = f(*planes, *planes_and_args[n_planes:])
    if isinstance(out, tuple):
        return tuple(np.swapaxes(o, 0, 1) for o in out)
    return np.swapaxes(out, 0, 1)


def dwt2(x, flt, transform: int, boundary: int, s: int = 1, real=None):
    """One level -> (aa, da, ad, dd): aa = lo_y(lo_x), da = lo_y(hi_x),
    ad = hi_y(lo_x), dd = hi_y(hi_x) (oracle.c's naming).  For the periodic
    variant `x` may be the unpadded plane of size real = (H, W) while the level
    works on its e_N padding to x-period (Hp, Wp) (R-24): pass x with
    x.shape == real and `real=(H, W, Hp, Wp)`."""
    lo, hi = flt[0], flt[1]
    if transform == 1:
        Lx, Hx = _along_x(dwt_swt, x, lo, hi, s)
        aa, ad = dwt_swt(Lx, lo, hi, s)
        da, dd = dwt_swt(Hx, lo, hi, s)
    elif boundary == 0:
        Lx, Hx = _along_x(dwt_sym, x, lo, hi)
        aa, ad = dwt_sym(Lx, lo, hi)
        da, dd = dwt_sym(Hx, lo, hi)
    else:
        H, W, Hp, Wp = real if real is not None else (x.shape[0], x.shape[1], x.shape[0], x.shape[1])
        Lx, Hx = _along_x(dwt_per, x, lo, hi, W, Wp)
        aa, ad = dwt_per(Lx, lo, hi, H, Hp)
        da, dd = dwt_per(Hx, lo, hi, H, Hp)
    return aa, da, ad, dd


def idwt2(aa, da, ad, dd, flt, transform: int, boundary: int, shape, s: int = 1):
    """Inverse of one level: columns first, then rows.  `shape` = (NH, NW) of the
    level's input plane (used by the expansive symmetric variant)."""
    lo, hi, rl, rh = flt
    if transform == 1:
        Lx = idwt_swt(aa, ad, lo, hi, s)
        Hx = idwt_swt(da, dd, lo, hi, s)
        return _along_x(idwt_swt, Lx, Hx, lo, hi, s, n_planes=2)
    if boundary == 0:
        NH, NW = shape
        Lx = idwt_sym(aa, ad, rl, rh, NH)
        Hx = idwt_sym(da, dd, rl, rh, NH)
        return _along_x(idwt_sym, Lx, Hx, rl, rh, NW, n_planes=2)
    Lx = idwt_per(aa, ad, lo, hi)
    Hx = idwt_per(da, dd, lo, hi)
    return _along_x(idwt_per, Lx, Hx, lo, hi, n_planes=2)


def padded_shape(H: int, W: int, levels: int):
    """R-24: H, W rounded up to multiples of 2^levels."""
    m = 1 << levels
    return -(-H // m) * m, -(-W // m) * m


# ------------------------------------------------------------------ denoiser / residual
def denoise(I, sigma0_sq: float = DEFAULT_SIGMA0_SQ, windows=DEFAULT_WINDOWS, levels: int = DEFAULT_LEVELS,
            taps: int = 8, boundary: int = 0, transform: int = 0, return_coeffs: bool = False):
    """F(I) in fp64 for one plane: decomposition, shrink of every detail subband
    (approximation passes through), inverse; cropped to H x W (R-24)."""
    x = np.asarray(I, dtype=np.float64)
    H, W = x.shape
    if H < (1 << levels) or W < (1 << levels):
        raise ValueError("PlaneTooSmall (S:116)")
    flt = filters_for(taps)
    per = transform == 0 and boundary == 1
    shapes, det = [], []
    cur = x
    for l in range(1, levels + 1):
        s = 1 << (l - 1)
        real = None
        if per and l == 1:
            real = (H, W) + padded_shape(H, W, levels)
            shapes.append(real[2:])
        else:
            shapes.append(cur.shape)
        aa, da, ad, dd = dwt2(cur, flt, transform, boundary, s=s, real=real)
        det.append(tuple(_shrink(c, sigma0_sq, windows) for c in (da, ad, dd)))
        cur = aa
    approx = cur
    for l in range(levels, 0, -1):
        da, ad, dd = det[l - 1]
        approx = idwt2(approx, da, ad, dd, flt, transform, boundary, shapes[l - 1], s=1 << (l - 1))
    return approx[:H, :W]


def residual(I, sigma0_sq: float = DEFAULT_SIGMA0_SQ, windows=DEFAULT_WINDOWS, levels: int = DEFAULT_LEVELS,
             taps: int = 8, boundary: int = 0, transform: int = 0, zero_mean: bool = False):
    """W = I - F(I) with the chosen variant; fp32 plane in, fp64 out."""
    x = np.asarray(I, dtype=np.float32).astype(np.float64)
    Wr = x - denoise(x, sigma0_sq, windows, levels, taps, boundary, transform)
    if zero_mean:
        Wr = _zero_mean(Wr)
    return Wr
