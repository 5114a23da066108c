"""oracle — plain fp64 CPU oracle for the SDA-frame PRNU hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_1909_04573_b200``) never imports it, and it
never imports the product path: the two share no code.

* a1-a6 (SDA mean, DWT, shrink, IDWT, MLE, finalize) live in ``oracle.c``
  (plain loops, fp64), loaded here through ctypes.
* a7-a8 (NCC, PCE) live in :mod:`oracle.match` (numpy fp64, ``numpy.fft``).
* f3 denoiser variants (db8, pad + periodic, undecimated) live in
  :mod:`oracle.variants` (numpy fp64, step by step; shrink from ``oracle.c``).

Citations: ``P:<n>`` PAPER.md line, ``S:<n>`` SPEC.md line, ``R-<n>`` a
reading listed in DESIGN.md.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

DEFAULT_SIGMA0_SQ = 9.0
DEFAULT_WINDOWS = (3, 5, 7, 9)
DEFAULT_LEVELS = 4
DEFAULT_EPS = 1e-6


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc, fp64, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fPIC", "-shared",
               "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        fp = ctypes.POINTER(ctypes.c_float)
        up = ctypes.POINTER(ctypes.c_uint8)
        ip = ctypes.POINTER(ctypes.c_int)
        L.oracle_sda_groups.argtypes = [ctypes.c_long, ctypes.c_long]
        L.oracle_sda_groups.restype = ctypes.c_long
        L.oracle_sda_average.argtypes = [up, ctypes.c_long, ctypes.c_int, ctypes.c_int, ctypes.c_long, fp]
        L.oracle_filters.argtypes = [dp, dp, dp, dp]
        L.oracle_ext.argtypes = [ctypes.c_long, ctypes.c_long]
        L.oracle_ext.restype = ctypes.c_int
        L.oracle_subband_len.argtypes = [ctypes.c_int]
        L.oracle_dwt1d.argtypes = [dp, ctypes.c_long, ctypes.c_int, dp, dp, ctypes.c_long]
        L.oracle_idwt1d.argtypes = [dp, dp, ctypes.c_long, ctypes.c_int, ctypes.c_int, dp, ctypes.c_long]
        L.oracle_dwt2d.argtypes = [dp, ctypes.c_int, ctypes.c_int, dp, dp, dp, dp]
        L.oracle_idwt2d.argtypes = [dp, dp, dp, dp, ctypes.c_int, ctypes.c_int, dp]
        L.oracle_box_mean_sq.argtypes = [dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, dp]
        L.oracle_shrink.argtypes = [dp, ctypes.c_int, ctypes.c_int, ctypes.c_double, ip, ctypes.c_int, dp]
        L.oracle_denoise.argtypes = [dp, ctypes.c_int, ctypes.c_int, ctypes.c_double, ip, ctypes.c_int,
                                     ctypes.c_int, dp]
        L.oracle_residual.argtypes = [fp, ctypes.c_int, ctypes.c_int, ctypes.c_double, ip, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_int, dp]
        L.oracle_mle_accumulate.argtypes = [dp, fp, ctypes.c_long, dp, dp]
        L.oracle_zero_mean.argtypes = [dp, ctypes.c_int, ctypes.c_int]
        L.oracle_finalize.argtypes = [dp, dp, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int, dp]
        L.oracle_extract_fingerprint.argtypes = [up, ctypes.c_long, ctypes.c_int, ctypes.c_int, ctypes.c_long,
                                                 ctypes.c_double, ip, ctypes.c_int, ctypes.c_int,
                                                 ctypes.c_double, ctypes.c_int, dp, dp, dp]
        for name in ("oracle_sda_average", "oracle_denoise", "oracle_residual", "oracle_extract_fingerprint"):
            getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"oracle {what} failed with status {code}")
        self.code = code


def _p(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _windows(windows):
    w = np.ascontiguousarray(np.asarray(windows, dtype=np.int32))
    return w, _p(w, ctypes.c_int)


# ---------------------------------------------------------------- a1
def sda_groups(m: int, d: int) -> int:
    """Number of SDA frames floor(m/d); -1 if d<1 or d>m."""
    return int(lib().oracle_sda_groups(m, d))


def sda_average(frames: np.ndarray, depth: int) -> np.ndarray:
    """uint8 [m,H,W] -> fp32 [floor(m/d),H,W]; mean of each group of d."""
    frames = np.ascontiguousarray(frames, dtype=np.uint8)
    m, H, W = frames.shape
    ns = sda_groups(m, depth)
    if ns < 0:
        raise OracleError(3, "sda_average (depth exceeds frames)")
    out = np.empty((ns, H, W), dtype=np.float32)
    st = lib().oracle_sda_average(_p(frames, ctypes.c_uint8), m, H, W, depth, _p(out, ctypes.c_float))
    if st:
        raise OracleError(st, "sda_average")
    return out


# ---------------------------------------------------------------- f4 luma
def rgb_to_luma(rgb: np.ndarray, layout: str = "planar", rounding: str = "fp32") -> np.ndarray:
    """BT.601 luma Y = 0.299 R + 0.587 G + 0.114 B (BASELINE config 3).

    Plain definition: the exact integer s = 299 R + 587 G + 114 B (Y = s / 1000
    exactly); "fp32" returns the correctly rounded fp32 of s / 1000 (an IEEE
    fp32 division of two exactly representable operands), "u8" rounds s / 1000
    half to even in integer arithmetic."""
    rgb = np.asarray(rgb, dtype=np.uint8)
    if layout == "planar":
        r, g, b = (rgb[:, k].astype(np.int64) for k in range(3))
    elif layout == "interleaved":
        r, g, b = (rgb[..., k].astype(np.int64) for k in range(3))
    else:
        raise ValueError(layout)
    s = 299 * r + 587 * g + 114 * b
    if rounding == "fp32":
        return s.astype(np.float32) / np.float32(1000.0)
    q, rem = np.divmod(s, 1000)
    q = q + ((rem > 500) | ((rem == 500) & (q % 2 == 1)))
    return q.astype(np.uint8)


# ---------------------------------------------------------------- a2-a4
def filters():
    """(dec_lo, dec_hi, rec_lo, rec_hi), each float64[8]."""
    out = [np.zeros(8) for _ in range(4)]
    lib().oracle_filters(*[_p(o, ctypes.c_double) for o in out])
    return tuple(out)


def ext(i: int, N: int) -> int:
    return int(lib().oracle_ext(i, N))


def subband_len(N: int) -> int:
    return int(lib().oracle_subband_len(N))


def dwt1d(x):
    x = _f64(x)
    N = x.shape[0]
    n = subband_len(N)
    a, d = np.empty(n), np.empty(n)
    lib().oracle_dwt1d(_p(x, ctypes.c_double), 1, N, _p(a, ctypes.c_double), _p(d, ctypes.c_double), 1)
    return a, d


def idwt1d(a, d, N: int):
    a, d = _f64(a), _f64(d)
    x = np.empty(N)
    lib().oracle_idwt1d(_p(a, ctypes.c_double), _p(d, ctypes.c_double), 1, a.shape[0], N,
                        _p(x, ctypes.c_double), 1)
    return x


def dwt2d(x):
    """One level: returns (aa, da, ad, dd) — see oracle.c for the naming."""
    x = _f64(x)
    NH, NW = x.shape
    nH, nW = subband_len(NH), subband_len(NW)
    outs = [np.empty((nH, nW)) for _ in range(4)]
    lib().oracle_dwt2d(_p(x, ctypes.c_double), NH, NW, *[_p(o, ctypes.c_double) for o in outs])
    return tuple(outs)


def idwt2d(aa, da, ad, dd, NH: int, NW: int):
    da, ad, dd = _f64(da), _f64(ad), _f64(dd)
    aa_p = None
    if aa is not None:
        aa = _f64(aa)
        aa_p = _p(aa, ctypes.c_double)
    x = np.empty((NH, NW))
    lib().oracle_idwt2d(aa_p, _p(da, ctypes.c_double), _p(ad, ctypes.c_double), _p(dd, ctypes.c_double),
                        NH, NW, _p(x, ctypes.c_double))
    return x


def wavedec2(x, levels: int = DEFAULT_LEVELS):
    """[aa_L, (da_L, ad_L, dd_L), ..., (da_1, ad_1, dd_1)] plus the level shapes."""
    cur = _f64(x)
    shapes = [cur.shape]
    details = []
    for _ in range(levels):
        aa, da, ad, dd = dwt2d(cur)
        details.append((da, ad, dd))
        cur = aa
        shapes.append(cur.shape)
    return cur, details, shapes


def waverec2(aa, details, shapes):
    cur = aa
    for l in range(len(details), 0, -1):
        da, ad, dd = details[l - 1]
        NH, NW = shapes[l - 1]
        cur = idwt2d(cur, da, ad, dd, NH, NW)
    return cur


def box_mean_sq(c, w: int):
    c = _f64(c)
    out = np.empty_like(c)
    lib().oracle_box_mean_sq(_p(c, ctypes.c_double), c.shape[0], c.shape[1], w, _p(out, ctypes.c_double))
    return out


def shrink(c, sigma0_sq: float = DEFAULT_SIGMA0_SQ, windows=DEFAULT_WINDOWS):
    """Denoised detail coefficients c * v/(v+sigma0^2)."""
    c = _f64(c)
    w, wp = _windows(windows)
    out = np.empty_like(c)
    lib().oracle_shrink(_p(c, ctypes.c_double), c.shape[0], c.shape[1], sigma0_sq, wp, len(w),
                        _p(out, ctypes.c_double))
    return out


def denoise(I, sigma0_sq: float = DEFAULT_SIGMA0_SQ, windows=DEFAULT_WINDOWS, levels: int = DEFAULT_LEVELS):
    """F(I) in fp64."""
    I = _f64(I)
    w, wp = _windows(windows)
    F = np.empty_like(I)
    st = lib().oracle_denoise(_p(I, ctypes.c_double), I.shape[0], I.shape[1], sigma0_sq, wp, len(w), levels,
                              _p(F, ctypes.c_double))
    if st:
        raise OracleError(st, "denoise")
    return F


def residual(I, sigma0_sq: float = DEFAULT_SIGMA0_SQ, windows=DEFAULT_WINDOWS, levels: int = DEFAULT_LEVELS,
             zero_mean: bool = False):
    """W = I - F(I) for one fp32 plane; fp64 result."""
    I = np.ascontiguousarray(I, dtype=np.float32)
    w, wp = _windows(windows)
    out = np.empty(I.shape, dtype=np.float64)
    st = lib().oracle_residual(_p(I, ctypes.c_float), I.shape[0], I.shape[1], sigma0_sq, wp, len(w), levels,
                               int(zero_mean), _p(out, ctypes.c_double))
    if st:
        raise OracleError(st, "residual")
    return out


# ---------------------------------------------------------------- a5-a6
def mle_accumulate(Wres, I, num, den):
    Wres = _f64(Wres)
    I = np.ascontiguousarray(I, dtype=np.float32)
    assert num.dtype == np.float64 and den.dtype == np.float64 and num.flags.c_contiguous
    lib().oracle_mle_accumulate(_p(Wres, ctypes.c_double), _p(I, ctypes.c_float), Wres.size,
                                _p(num, ctypes.c_double), _p(den, ctypes.c_double))


def zero_mean(x):
    x = _f64(x).copy()
    lib().oracle_zero_mean(_p(x, ctypes.c_double), x.shape[0], x.shape[1])
    return x


def finalize(num, den, eps: float = DEFAULT_EPS, zero_mean: bool = True):
    num, den = _f64(num), _f64(den)
    K = np.empty_like(num)
    lib().oracle_finalize(_p(num, ctypes.c_double), _p(den, ctypes.c_double), num.shape[0], num.shape[1], eps,
                          int(zero_mean), _p(K, ctypes.c_double))
    return K


def extract_fingerprint(frames, depth: int, sigma0_sq: float = DEFAULT_SIGMA0_SQ, windows=DEFAULT_WINDOWS,
                        levels: int = DEFAULT_LEVELS, eps: float = DEFAULT_EPS, zero_mean: bool = True):
    """Returns (K fp64 [H,W], num, den, n_sda)."""
    frames = np.ascontiguousarray(frames, dtype=np.uint8)
    m, H, W = frames.shape
    w, wp = _windows(windows)
    K = np.empty((H, W))
    num = np.empty((H, W))
    den = np.empty((H, W))
    st = lib().oracle_extract_fingerprint(_p(frames, ctypes.c_uint8), m, H, W, depth, sigma0_sq, wp, len(w),
                                          levels, eps, int(zero_mean), _p(K, ctypes.c_double),
                                          _p(num, ctypes.c_double), _p(den, ctypes.c_double))
    if st:
        raise OracleError(st, "extract_fingerprint")
    return K, num, den, sda_groups(m, depth)


from .match import ncc, pce, correlation_surface, pce_template, block_grid, blockwise_match, wiener_dft  # noqa: E402,F401
