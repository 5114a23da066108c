"""Pins for the oracle's wavelet transform (a2, a4): filters, 1-D/2-D analysis
and synthesis.  Readings R-2 (8-tap Daubechies), R-4 (half-sample symmetric
extension), R-5 (phase/offset), R-6 (row/column order)."""
import math

import numpy as np
import pytest

import oracle


def daubechies_minphase(p: int) -> np.ndarray:
    """Independent spectral factorisation of the Daubechies polynomial.

    |H(w)|^2 = 2 cos^{2p}(w/2) P(sin^2(w/2)),  P(y) = sum_{k<p} C(p-1+k, k) y^k.
    With y = (2 - z - 1/z)/4 each root y_i of P gives z^2 - (2-4 y_i) z + 1 = 0;
    keep the root inside the unit circle (minimum phase)."""
    coeffs = [math.comb(p - 1 + k, k) for k in range(p)]       # ascending powers of y
    yroots = np.roots(coeffs[::-1])
    zroots = []
    for yi in yroots:
        zz = np.roots([1.0, -(2.0 - 4.0 * yi), 1.0])
        zroots.append(zz[np.argmin(np.abs(zz))])
    q = np.real(np.poly(zroots))
    h = q
    for _ in range(p):
        h = np.convolve(h, [1.0, 1.0])
    return h * (math.sqrt(2.0) / h.sum())


def test_filter_is_db4_minimum_phase_reversed():
    dec_lo, dec_hi, rec_lo, rec_hi = oracle.filters()
    h = daubechies_minphase(4)
    # R-2/R-5: rec_lo is the minimum-phase factor, dec_lo its time reverse
    np.testing.assert_allclose(rec_lo, h, atol=1e-12)
    np.testing.assert_allclose(dec_lo, h[::-1], atol=1e-12)


def test_filter_closed_forms():
    dec_lo, dec_hi, rec_lo, rec_hi = oracle.filters()
    assert abs(dec_lo.sum() - math.sqrt(2)) < 1e-14
    assert abs((dec_lo ** 2).sum() - 1) < 1e-14
    for j in (1, 2, 3):                                # double-shift orthogonality
        assert abs(np.dot(dec_lo[: 8 - 2 * j], dec_lo[2 * j:])) < 1e-14
    k = np.arange(8, dtype=np.float64)
    for q in range(4):                                  # 4 vanishing moments
        assert abs((k ** q * dec_hi).sum()) < 1e-11
    assert abs(np.dot(dec_lo, dec_hi)) < 1e-15          # lo/hi orthogonal
    np.testing.assert_allclose(rec_lo, dec_lo[::-1])
    np.testing.assert_allclose(rec_hi, dec_hi[::-1])


def test_extension_map():
    # R-4 half-sample symmetric: ... x1 x0 | x0 x1 ... x_{N-1} | x_{N-1} x_{N-2} ...
    N = 5
    got = [oracle.ext(i, N) for i in range(-7, N + 7)]
    xp = np.pad(np.arange(N), 7, mode="symmetric")        # numpy's definition
    assert got == [int(v) for v in xp]
    assert [oracle.ext(i, 1) for i in range(-3, 4)] == [0] * 7


def _np_analysis(x, f):
    """numpy formulation: pad 7 with mode='symmetric', 'valid' convolution, odd phase."""
    return np.convolve(np.pad(x, 7, mode="symmetric"), f, mode="valid")[1::2]


def _np_synthesis(a, d, N, rl, rh):
    """numpy formulation: zero-upsample, full convolution, keep [6, 6+N)."""
    n = a.size
    ua = np.zeros(2 * n - 1)
    ud = np.zeros(2 * n - 1)
    ua[::2] = a
    ud[::2] = d
    y = np.convolve(ua, rl) + np.convolve(ud, rh)
    return y[6: 6 + N]


@pytest.mark.parametrize("N", list(range(2, 41)) + [64, 135, 543, 1080])
def test_dwt1d_matches_numpy_convolution(N):
    rng = np.random.default_rng(N)
    x = rng.uniform(0, 255, N)
    dec_lo, dec_hi, rec_lo, rec_hi = oracle.filters()
    a, d = oracle.dwt1d(x)
    assert a.size == (N + 7) // 2
    np.testing.assert_allclose(a, _np_analysis(x, dec_lo), atol=1e-11)
    np.testing.assert_allclose(d, _np_analysis(x, dec_hi), atol=1e-11)
    np.testing.assert_allclose(oracle.idwt1d(a, d, N), _np_synthesis(a, d, N, rec_lo, rec_hi), atol=1e-11)


@pytest.mark.parametrize("N", list(range(2, 41)) + [135, 963, 1920])
def test_dwt1d_perfect_reconstruction(N):
    rng = np.random.default_rng(1000 + N)
    x = rng.uniform(0, 255, N)
    a, d = oracle.dwt1d(x)
    assert np.abs(oracle.idwt1d(a, d, N) - x).max() < 1e-10


@pytest.mark.parametrize("shape,levels", [((8, 8), 3), ((16, 16), 4), ((64, 64), 4), ((37, 53), 4),
                                          ((135, 240), 4), ((16, 200), 4), ((1080, 1920), 4)])
def test_wavedec2_perfect_reconstruction(shape, levels):
    """BASELINE north_star: DWT followed by IDWT reconstructs to 1e-10."""
    rng = np.random.default_rng(shape[0] * 7 + shape[1])
    x = rng.uniform(0, 255, shape)
    aa, det, shapes = oracle.wavedec2(x, levels)
    assert np.abs(oracle.waverec2(aa, det, shapes) - x).max() < 1e-10


def test_subband_sizes_fhd():
    # S-8(a) table: 1080x1920 -> 543x963, 275x485, 141x246, 74x126
    _, det, shapes = oracle.wavedec2(np.zeros((1080, 1920)), 4)
    assert shapes[1:] == [(543, 963), (275, 485), (141, 246), (74, 126)]


def test_constant_plane_closed_form():
    """Symmetric extension of a constant is constant: aa = 2c (sum(h)^2 = 2),
    every detail coefficient is 0 (zeroth vanishing moment)."""
    c = 93.25
    aa, da, ad, dd = oracle.dwt2d(np.full((21, 34), c))
    np.testing.assert_allclose(aa, 2 * c, rtol=1e-14)
    for s in (da, ad, dd):
        assert np.abs(s).max() < 1e-12


def test_cubic_polynomial_interior_details_vanish():
    """4 vanishing moments: details of a cubic vanish away from the borders."""
    N = 64
    t = np.arange(N, dtype=np.float64)
    x = 0.001 * t ** 3 - 0.05 * t ** 2 + 2 * t + 7
    a, d = oracle.dwt1d(x)
    interior = slice(4, (N + 7) // 2 - 4)
    assert np.abs(d[interior]).max() < 1e-9
    assert np.abs(d).max() > 1e-3           # but not at the (mirrored) borders


def test_separable_2d_equals_matrix_form():
    """2-D level == A_y X A_x^T with the 1-D analysis matrices (built from numpy)."""
    rng = np.random.default_rng(3)
    NH, NW = 13, 22
    X = rng.uniform(0, 255, (NH, NW))
    dec_lo, dec_hi, _, _ = oracle.filters()

    def mat(N, f):
        return np.stack([_np_analysis(e, f) for e in np.eye(N)], axis=1)

    AyL, AyH, AxL, AxH = mat(NH, dec_lo), mat(NH, dec_hi), mat(NW, dec_lo), mat(NW, dec_hi)
    aa, da, ad, dd = oracle.dwt2d(X)
    np.testing.assert_allclose(aa, AyL @ X @ AxL.T, atol=1e-10)
    np.testing.assert_allclose(da, AyL @ X @ AxH.T, atol=1e-10)   # high-pass along x
    np.testing.assert_allclose(ad, AyH @ X @ AxL.T, atol=1e-10)   # high-pass along y
    np.testing.assert_allclose(dd, AyH @ X @ AxH.T, atol=1e-10)
