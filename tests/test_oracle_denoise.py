"""Pins for the oracle's shrink (a3) and residual W = I - F(I) (a4): P:83,
P:150; readings R-1..R-8."""
import numpy as np
import pytest
from scipy import ndimage

import oracle

from test_oracle_wavelet import _np_analysis, _np_synthesis


@pytest.mark.parametrize("shape", [(7, 7), (10, 14), (3, 5), (2, 2), (1, 4), (35, 21), (4, 9)])
@pytest.mark.parametrize("w", [3, 5, 7, 9])
def test_box_mean_matches_scipy_reflect(shape, w):
    """R-7: mirror windows of w^2 samples == scipy uniform_filter(mode='reflect')."""
    rng = np.random.default_rng(w * 100 + shape[0])
    c = rng.normal(0, 5, shape)
    ref = ndimage.uniform_filter(c * c, size=w, mode="reflect")
    np.testing.assert_allclose(oracle.box_mean_sq(c, w), ref, atol=1e-12, rtol=1e-12)


def test_shrink_isolated_spike_closed_form():
    """Single spike a at an interior point: every window's mean of c^2 is a^2/w^2,
    the minimum is the 9x9 one, v = max(0, a^2/81 - 9); c_hat = a v/(v+9);
    all other coefficients are 0 and stay 0."""
    a = 60.0
    c = np.zeros((21, 21))
    c[10, 10] = a
    out = oracle.shrink(c, 9.0, (3, 5, 7, 9))
    v = a * a / 81.0 - 9.0
    assert abs(out[10, 10] - a * v / (v + 9.0)) < 1e-12
    out[10, 10] = 0
    assert np.abs(out).max() == 0.0


def test_shrink_corner_spike_mirror():
    """Spike at (0,0): half-sample mirroring repeats it twice per axis in every
    window, so the 9x9 mean is 4 a^2 / 81."""
    a = 30.0
    c = np.zeros((12, 12))
    c[0, 0] = a
    out = oracle.shrink(c, 9.0, (3, 5, 7, 9))
    v = 4 * a * a / 81.0 - 9.0
    assert abs(out[0, 0] - a * v / (v + 9.0)) < 1e-12


def test_shrink_below_noise_floor_is_zero_and_constant_case():
    c = np.full((9, 9), 2.0)          # c^2 = 4 < sigma0^2 -> v = 0 -> fully attenuated
    assert np.abs(oracle.shrink(c)).max() == 0.0
    c = np.full((9, 9), 5.0)          # v = 25 - 9 = 16 -> 5 * 16/25 = 3.2
    np.testing.assert_allclose(oracle.shrink(c), 3.2, rtol=1e-15)


def test_shrink_limits():
    rng = np.random.default_rng(1)
    c = rng.normal(0, 10, (15, 15))
    np.testing.assert_allclose(oracle.shrink(c, 1e-12), c, rtol=1e-9)  # sigma0 -> 0: identity
    assert np.abs(oracle.shrink(c, 1e12)).max() < 1e-9                  # sigma0 -> inf: zero


def _tex(shape, seed):
    rng = np.random.default_rng(seed)
    y, x = np.mgrid[0: shape[0], 0: shape[1]]
    I = 128 + 40 * np.sin(2 * np.pi * x / 23.0) * np.cos(2 * np.pi * y / 17.0) + rng.normal(0, 3, shape)
    return np.round(np.clip(I, 0, 245)).astype(np.float32)   # integers: I + 10 is exact in fp32


def test_constant_plane_zero_residual():
    """S:120, BASELINE: a constant image gives a zero residual."""
    for shape in [(64, 64), (37, 53), (16, 16)]:
        W = oracle.residual(np.full(shape, 128.0, np.float32))
        assert np.abs(W).max() < 1e-10


def test_offset_invariance():
    """W(I + c) == W(I)."""
    I = _tex((48, 80), 0)
    d = oracle.residual(I + np.float32(10.0)) - oracle.residual(I)
    assert np.abs(d).max() < 1e-10


def test_transpose_covariance():
    I = _tex((45, 61), 1)
    d = oracle.residual(np.ascontiguousarray(I.T)) - oracle.residual(I).T
    assert np.abs(d).max() < 1e-10


def test_homogeneity():
    """The Wiener rule is scale-covariant: W(aI; a^2 s0) = a W(I; s0)."""
    I = _tex((40, 40), 2)
    a = 2.0  # exact in fp32
    d = oracle.residual(I * np.float32(a), sigma0_sq=9.0 * a * a) - a * oracle.residual(I, 9.0)
    assert np.abs(d).max() < 1e-9


def test_sigma_limits():
    I = _tex((32, 48), 3)
    # sigma0 -> inf: every detail is removed, W = I - IDWT(approximation only)
    aa, det, shapes = oracle.wavedec2(I.astype(np.float64), 4)
    zero = [tuple(np.zeros_like(s) for s in lvl) for lvl in det]
    proj = oracle.waverec2(aa, zero, shapes)
    np.testing.assert_allclose(oracle.residual(I, sigma0_sq=1e30), I - proj, atol=1e-9)
    # sigma0 -> 0: nothing is removed, W -> 0
    assert np.abs(oracle.residual(I, sigma0_sq=1e-12)).max() < 1e-6


def test_white_noise_attenuation():
    """white noise sigma=3, sigma0^2 = 9 -> var(F(I)) < 0.25 var(I), 20 seeds."""
    ratios = []
    for s in range(20):
        rng = np.random.default_rng(s)
        I = rng.normal(0, 3, (64, 64))
        F = oracle.denoise(I)
        ratios.append(F.var() / I.var())
    assert max(ratios) < 0.25


def test_impulse():
    """constant 128 + impulse of +50 at the centre -> F(centre) strictly in (128, 178)."""
    I = np.full((64, 64), 128.0)
    I[32, 32] += 50
    F = oracle.denoise(I)
    assert 128.0 < F[32, 32] < 178.0


def test_plane_too_small():
    with pytest.raises(oracle.OracleError) as e:
        oracle.residual(np.zeros((15, 64), np.float32))
    assert e.value.code == 2   # S:116-118 PlaneTooSmall


def test_brute_force_8x8_matrix_denoiser():
    """North star: brute force on 8x8 (L = 3, 2^3 = 8).  Build every level from
    explicit analysis/synthesis matrices (numpy pad/convolve formulation),
    shrink with scipy uniform_filter, and compare W with the oracle."""
    dec_lo, dec_hi, rec_lo, rec_hi = oracle.filters()

    def amat(N, f):
        return np.stack([_np_analysis(e, f) for e in np.eye(N)], axis=1)

    def smat(n, N):
        lo = np.stack([_np_synthesis(e, np.zeros(n), N, rec_lo, rec_hi) for e in np.eye(n)], axis=1)
        hi = np.stack([_np_synthesis(np.zeros(n), e, N, rec_lo, rec_hi) for e in np.eye(n)], axis=1)
        return lo, hi

    def shrink_ref(c):
        est = np.full(c.shape, np.inf)
        for w in (3, 5, 7, 9):
            est = np.minimum(est, np.maximum(0.0, ndimage.uniform_filter(c * c, w, mode="reflect") - 9.0))
        return c * est / (est + 9.0)

    rng = np.random.default_rng(8)
    X0 = rng.integers(0, 256, (8, 8)).astype(np.float32)
    X = X0.astype(np.float64)
    levels = 3
    Ns = [8]
    cur = X
    dets = []
    for _ in range(levels):
        N = cur.shape[0]
        AL, AH = amat(N, dec_lo), amat(N, dec_hi)
        dets.append((AL @ cur @ AH.T, AH @ cur @ AL.T, AH @ cur @ AH.T))
        cur = AL @ cur @ AL.T
        Ns.append(cur.shape[0])
    for l in range(levels, 0, -1):
        da, ad, dd = (shrink_ref(s) for s in dets[l - 1])
        N, n = Ns[l - 1], Ns[l]
        SL, SH = smat(n, N)
        cur = SL @ cur @ SL.T + SL @ da @ SH.T + SH @ ad @ SL.T + SH @ dd @ SH.T
    W_ref = X - cur
    W = oracle.residual(X0, levels=levels)
    np.testing.assert_allclose(W, W_ref, atol=1e-10)
