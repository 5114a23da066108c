"""Pins of the f3 denoiser-variant oracle (oracle/variants.py) against what the
mathematics fixes: filter closed forms, perfect reconstruction, Parseval / the
tight-frame bound, explicit matrices, numpy's own symmetric padding, the C
oracle for the default variant, and the denoiser invariants of S:120-S:143."""
import numpy as np
import pytest

import oracle
from oracle import variants as V

VARIANTS = [dict(taps=8, boundary=0, transform=0), dict(taps=16, boundary=0, transform=0),
            dict(taps=8, boundary=1, transform=0), dict(taps=16, boundary=1, transform=0),
            dict(taps=8, boundary=0, transform=1), dict(taps=16, boundary=0, transform=1)]


def _rng(seed):
    return np.random.default_rng(seed)


# ------------------------------------------------------------------ filters (Q2)
def test_db4_spectral_factorisation_reproduces_typed_dec_lo():
    """The factorisation at p = 4 equals oracle.c's typed DEC_LO (itself pinned by
    its closed-form properties in test_oracle_pins)."""
    lo = oracle.filters()[0]
    assert np.abs(V.daubechies(4) - lo).max() < 1e-14


@pytest.mark.parametrize("p", [4, 8])
def test_daubechies_closed_form_properties(p):
    h = V.daubechies(p)
    L = 2 * p
    assert len(h) == L
    assert abs(h.sum() - np.sqrt(2.0)) < 1e-14                    # lowpass DC gain sqrt(2)
    assert abs((h * h).sum() - 1.0) < 1e-14                       # unit norm
    for j in range(1, p):                                         # orthogonal to its even shifts
        assert abs(np.dot(h[2 * j:], h[:L - 2 * j])) < 1e-14
    g = V.qmf(h)[1]
    k = np.arange(L, dtype=np.float64)
    for m in range(p):                                            # p vanishing moments of the highpass
        assert abs(np.sum(k ** m * g)) <= 1e-12 * np.sum(k ** m * np.abs(g))
    # minimum phase (Daubechies' root choice): rec_lo = reverse(dec_lo) has all
    # zeros other than the p-fold zero at z = -1 strictly inside the unit circle
    # (the p-fold root is ill-conditioned, so divide it out exactly first)
    q = h[::-1].copy()
    for _ in range(p):
        q, rem = np.polydiv(q, [1.0, 1.0])
        assert np.abs(rem).max() < 1e-12                          # (1 + z) divides: the p-fold zero
    r = np.roots(q)
    assert len(r) == p - 1 and np.abs(r).max() < 1.0


def test_db8_is_not_db4_padded():
    """A dropped-term guard: db8 has 16 non-negligible taps."""
    h = V.daubechies(8)
    assert np.abs(h).min() > 1e-5 and abs(h[0]) < 1e-3 and abs(h[-1]) > 0.05


# ------------------------------------------------------------------ perfect reconstruction
@pytest.mark.parametrize("taps", [8, 16])
@pytest.mark.parametrize("N", [1, 2, 5, 8, 9, 16, 17, 35, 64])
def test_sym_pr(taps, N):
    lo, hi, rl, rh = V.filters_for(taps)
    x = _rng(N).uniform(0, 255, (N, 3))
    a, d = V.dwt_sym(x, lo, hi)
    assert a.shape[0] == (N + taps - 1) // 2
    assert np.abs(V.idwt_sym(a, d, rl, rh, N) - x).max() < 1e-10


@pytest.mark.parametrize("taps", [8, 16])
@pytest.mark.parametrize("N", [2, 4, 8, 16, 18, 64])
def test_per_pr_and_parseval(taps, N):
    lo, hi, _, _ = V.filters_for(taps)
    x = _rng(N + 1).uniform(0, 255, (N, 2))
    a, d = V.dwt_per(x, lo, hi)
    assert a.shape[0] == N // 2
    assert np.abs(V.idwt_per(a, d, lo, hi) - x).max() < 1e-10
    e = (a * a).sum() + (d * d).sum()
    assert abs(e - (x * x).sum()) <= 1e-13 * (x * x).sum()        # orthogonal: Parseval


@pytest.mark.parametrize("taps", [8, 16])
@pytest.mark.parametrize("N,s", [(1, 1), (3, 2), (16, 1), (16, 8), (17, 4), (40, 8)])
def test_swt_pr_and_frame_bound(taps, N, s):
    lo, hi, _, _ = V.filters_for(taps)
    x = _rng(N * s).uniform(0, 255, (N, 2))
    a, d = V.dwt_swt(x, lo, hi, s)
    assert np.abs(V.idwt_swt(a, d, lo, hi, s) - x).max() < 1e-10
    e = (a * a).sum() + (d * d).sum()
    assert abs(e - 2 * (x * x).sum()) <= 1e-13 * (x * x).sum()    # tight frame, bound 2


def _matrix(f, N):
    cols = []
    for i in range(N):
        e = np.zeros((N, 1))
        e[i] = 1.0
        a, d = f(e)
        cols.append(np.concatenate([a[:, 0], d[:, 0]]))
    return np.stack(cols, axis=1)


def test_explicit_matrices():
    """Brute force: the periodic analysis matrix is orthogonal (A^T A = I) and the
    undecimated one is a tight frame (A^T A = 2 I), at 16 taps and N = 16."""
    lo, hi, _, _ = V.filters_for(16)
    A = _matrix(lambda e: V.dwt_per(e, lo, hi), 16)
    assert A.shape == (16, 16) and np.abs(A.T @ A - np.eye(16)).max() < 1e-13
    S = _matrix(lambda e: V.dwt_swt(e, lo, hi, 2), 16)
    assert S.shape == (32, 16) and np.abs(S.T @ S - 2 * np.eye(16)).max() < 1e-13


# ------------------------------------------------------------------ 2-D residuals
def test_default_variant_equals_c_oracle():
    """taps 8, symmetric, decimated through the numpy variant code == oracle.c."""
    for H, W, lv in [(37, 53, 4), (64, 64, 4), (16, 40, 3)]:
        I = _rng(H * W).uniform(0, 255, (H, W)).astype(np.float32)
        assert np.abs(V.residual(I, levels=lv) - oracle.residual(I, levels=lv)).max() < 1e-10


@pytest.mark.parametrize("taps", [8, 16])
def test_periodic_padding_equals_numpy_symmetric_pad(taps):
    """R-24: the implicit e_N padding equals numpy.pad(mode='symmetric') followed by
    the periodic denoiser on the padded plane, cropped."""
    H, W, lv = 37, 53, 3
    I = _rng(7).uniform(0, 255, (H, W))
    Hp, Wp = V.padded_shape(H, W, lv)
    assert (Hp, Wp) == (40, 56)
    Ip = np.pad(I, ((0, Hp - H), (0, Wp - W)), mode="symmetric")
    a = V.denoise(I, levels=lv, taps=taps, boundary=1)
    b = V.denoise(Ip, levels=lv, taps=taps, boundary=1)[:H, :W]
    assert np.abs(a - b).max() < 1e-10


@pytest.mark.parametrize("kw", VARIANTS)
def test_variant_invariants(kw):
    H, W = 40, 56
    g = _rng(3)
    y, x = np.mgrid[0:H, 0:W]
    I = np.round(128 + 60 * np.sin(x / 5.0 + y / 7.0) + g.normal(0, 5, (H, W))).astype(np.float32)   # exact +17, *2
    Wr = V.residual(I, **kw)
    assert np.abs(V.residual(np.full((H, W), 93.0, np.float32), **kw)).max() < 1e-10
    assert np.abs(V.residual(I + 17.0, **kw) - Wr).max() < 1e-9
    assert np.abs(V.residual(I.T.copy(), **kw) - Wr.T).max() < 1e-9                   # transpose
    a = 2.0                                                                            # homogeneity
    Wa = V.residual((I.astype(np.float64) * a), sigma0_sq=9.0 * a * a, **kw)
    assert np.abs(Wa - a * Wr).max() < 1e-8
    assert np.abs(V.residual(I, sigma0_sq=1e-30, **kw)).max() < 1e-8                 # sigma0^2 -> 0


@pytest.mark.parametrize("kw", VARIANTS)
def test_variant_white_noise_suppression(kw):
    """on white noise of variance sigma0^2 the denoised output keeps < 25 % of the variance."""
    n = _rng(11).normal(0, 3.0, (64, 64))
    F = V.denoise(128.0 + n, **kw) - 128.0
    assert F.var() / n.var() < 0.25


def test_variants_differ_from_default():
    """Each variant is a different denoiser (guards against a silently ignored option)."""
    I = _rng(5).uniform(0, 255, (40, 56)).astype(np.float32)
    base = V.residual(I)
    for kw in VARIANTS[1:]:
        assert np.abs(V.residual(I, **kw) - base).max() > 1e-3, kw
