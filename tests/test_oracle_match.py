"""Pins for the oracle's NCC (a7) and PCE (a8): P:93; S:284-331;
readings R-15..R-20."""
import numpy as np
import pytest

import oracle
from oracle import match


def brute_surface(R, T):
    """Direct O(N^4) circular correlation of the mean-removed inputs."""
    R = R - R.mean()
    T = T - T.mean()
    H, W = R.shape
    C = np.zeros((H, W))
    for dy in range(H):
        for dx in range(W):
            C[dy, dx] = np.sum(R * np.roll(T, (dy, dx), axis=(0, 1)))
    return C


@pytest.mark.parametrize("shape", [(8, 8), (13, 21), (32, 32)])
def test_fft_surface_equals_brute_force(shape):
    """S:292, S:322 (AC7): FFT surface == direct spatial computation."""
    rng = np.random.default_rng(shape[0])
    R, T = rng.normal(size=shape), rng.normal(size=shape)
    np.testing.assert_allclose(oracle.correlation_surface(R, T), brute_surface(R, T), atol=1e-9)


def test_shift_theorem_and_peak():
    """R = T circularly shifted by (3, 5) -> peak at (3, 5)."""
    rng = np.random.default_rng(0)
    T = rng.normal(size=(40, 48))
    R = np.roll(T, (3, 5), axis=(0, 1))
    p, (dy, dx), peak = oracle.pce(R, T)
    assert (dy, dx) == (3, 5)
    assert p > 1e3
    p2, shift2, _ = oracle.pce(np.roll(R, (7, 1), axis=(0, 1)), T)
    assert shift2 == (10, 6)
    assert abs(p2 - p) / p < 1e-9


def test_scale_invariance():
    """positive gains leave PCE unchanged."""
    rng = np.random.default_rng(1)
    R, T = rng.normal(size=(32, 32)), rng.normal(size=(32, 32))
    R[0, 0] += 20
    T[0, 0] += 20
    a = oracle.pce(R, T)[0]
    b = oracle.pce(3.5 * R + 2.0, 0.25 * T - 7.0)[0]
    assert abs(a - b) / abs(a) < 1e-9


def test_pce_closed_form_surface():
    """Surface with C[2,3] = 10 and 1 elsewhere: the 11x11 neighbourhood holds 120
    ones, background mean of C^2 = (255 - 120)/(256 - 121) = 1 -> PCE = 100."""
    C = np.ones((16, 16))
    C[2, 3] = 10.0
    p, peak, v = match.pce_from_surface(C, 5)
    assert peak == (2, 3) and v == 10.0
    assert abs(p - 100.0) < 1e-12
    C[2, 3] = -10.0                          # sign is kept
    assert abs(match.pce_from_surface(C, 5)[0] + 100.0) < 1e-12


def test_delta_surface_caps():
    """delta surface -> zero background energy -> cap 1e12."""
    C = np.zeros((16, 16))
    C[0, 0] = 1.0
    assert match.pce_from_surface(C, 5)[0] == match.PCE_CAP


def test_argmax_tie_smallest_index():
    C = np.zeros((20, 20))
    C[3, 4] = -2.0
    C[1, 7] = 2.0
    C[15, 15] = 0.5
    assert match.pce_from_surface(C, 2)[1] == (1, 7)


def test_null_calibration():
    """S:300, S:608 (AC8): independent random inputs -> P(PCE > 60) < 5%."""
    rng = np.random.default_rng(7)
    hits = 0
    for _ in range(200):
        R, T = rng.normal(size=(128, 128)), rng.normal(size=(128, 128))
        hits += oracle.pce(R, T)[0] > match.PCE_THRESHOLD
    assert hits / 200 < 0.05


def test_ncc_properties():
    rng = np.random.default_rng(2)
    a = rng.normal(size=(20, 30))
    assert abs(oracle.ncc(a, a) - 1) < 1e-15
    assert abs(oracle.ncc(a, -a) + 1) < 1e-15
    assert abs(oracle.ncc(a, 3 * a + 7) - 1) < 1e-14
    assert abs(oracle.ncc(a, -0.5 * a + 1) + 1) < 1e-14
    b = rng.normal(size=(20, 30))
    # equals the value of the correlation surface at shift 0 normalised by the norms
    C = oracle.correlation_surface(a, b)
    a0, b0 = a - a.mean(), b - b.mean()
    assert abs(C[0, 0] / np.sqrt((a0 ** 2).sum() * (b0 ** 2).sum()) - oracle.ncc(a, b)) < 1e-14
    with pytest.raises(ValueError):
        oracle.ncc(np.ones((4, 4)), a[:4, :4])


def test_aligned_pce_uses_origin():
    rng = np.random.default_rng(3)
    T = rng.normal(size=(32, 32))
    R = np.roll(T, (4, 4), axis=(0, 1))
    p_al, peak, _ = oracle.pce(R, T, aligned=True)
    assert peak == (0, 0)
    assert p_al < oracle.pce(R, T)[0]


def test_threshold_strict():
    """pce exactly 60 -> no match (strict '>')."""
    assert not (60.0 > match.PCE_THRESHOLD)


def test_block_grid_spec_examples():
    """1000x500 frame, block 500 -> 2 tiles; 1024x512 -> edge tiles kept."""
    g = match.block_grid(500, 1000, 500)      # H=500 rows, W=1000 cols
    assert g == [(0, 0, 500, 500), (0, 500, 500, 500)]
    g = match.block_grid(512, 1024, 500)
    assert len(g) == 6 and (0, 1000, 500, 24) in g and (500, 1000, 12, 24) in g
    assert sum(h * w for (_, _, h, w) in g) == 512 * 1024             # disjoint cover
    assert len(match.block_grid(1000, 1000, 500)) == 4


def test_blockwise_equals_per_tile_aligned_pce():
    rng = np.random.default_rng(9)
    T = rng.normal(size=(70, 90))
    R = 0.3 * T + rng.normal(size=T.shape)
    res = match.blockwise_match(R, T, block=32)
    assert len(res) == 3 * 3
    for (y, x, h, w, p, c) in res:
        r, t = R[y:y + h, x:x + w], T[y:y + h, x:x + w]
        C = brute_surface(r, t)                       # direct correlation of the tile
        pp = match.pce_from_surface(C, 5, peak=(0, 0))[0]
        assert abs(p - pp) <= 1e-9 * abs(pp)
        assert abs(c - oracle.ncc(r, t)) < 1e-12
        assert p > 0 and c > 0.1                      # matched tiles correlate


# ---------------------------------------------------------------- f2: Wiener filtering in the DFT domain (R-23)
def test_wdft_delta_is_fixed_point():
    """A unit impulse has a flat magnitude spectrum: A^2 = 1/(HW) = s2 everywhere,
    so every box mean equals s2 and the gain s2/max(m, s2) is exactly 1."""
    K = np.zeros((16, 24))
    K[3, 5] = 1.0
    assert np.max(np.abs(oracle.wiener_dft(K) - K)) < 1e-12


def test_wdft_homogeneous_and_real():
    rng = np.random.default_rng(1)
    K = rng.normal(0, 0.01, (20, 28))
    K -= K.mean()
    a = oracle.wiener_dft(K)
    assert np.max(np.abs(oracle.wiener_dft(3.5 * K) - 3.5 * a)) < 1e-12   # gain is scale-free
    assert np.isrealobj(a) and abs(a.mean()) < 1e-12                     # zero-mean stays zero-mean


def test_wdft_attenuates_a_periodic_component_not_the_noise():
    """A strong periodic pattern (a spectral peak, the artefact WDFT targets) is
    attenuated; the white part passes with gain <= 1 and keeps most of its energy."""
    rng = np.random.default_rng(2)
    H, W = 64, 64
    noise = rng.normal(0, 0.01, (H, W))
    y, x = np.mgrid[0:H, 0:W]
    periodic = 0.05 * np.cos(2 * np.pi * (5 * y / H + 9 * x / W))
    K = noise + periodic
    K -= K.mean()
    out = oracle.wiener_dft(K)
    def peak(z):
        return np.abs(np.fft.fft2(z))[5, 9]
    assert peak(out) < 0.2 * peak(K)
    rest = out - (np.sum(out * periodic) / np.sum(periodic * periodic)) * periodic
    assert 0.5 * np.sum(noise ** 2) < np.sum(rest ** 2) <= 1.01 * np.sum(noise ** 2)


def test_wdft_gain_matches_brute_force_windows():
    """The box means inside wiener_dft use scipy 'reflect' = the e_N mirror windows
    (R-7): brute force on a tiny plane."""
    rng = np.random.default_rng(3)
    K = rng.normal(0, 1, (5, 6))
    K -= K.mean()
    H, W = K.shape
    F = np.fft.fft2(K)
    A2 = np.abs(F) ** 2 / (H * W)
    s2 = np.mean(K * K)
    def e(i, N):
        r = i % (2 * N)
        return r if r < N else 2 * N - 1 - r
    m = np.full((H, W), np.inf)
    for w in (3, 5, 7, 9):
        h = w // 2
        box = np.array([[np.mean([A2[e(u + dy, H), e(v + dx, W)] for dy in range(-h, h + 1)
                                  for dx in range(-h, h + 1)]) for v in range(W)] for u in range(H)])
        m = np.minimum(m, box)
    ref = np.real(np.fft.ifft2(F * (s2 / np.maximum(m, s2))))
    assert np.max(np.abs(oracle.wiener_dft(K) - ref)) < 1e-12


def _cos(H, W, c, fy, fx):
    y, x = np.mgrid[0:H, 0:W]
    return c * np.cos(2 * np.pi * (fy * y / H + fx * x / W))


def test_wdft_closed_form_isolated_cosines():
    """R-23 in closed form, without the oracle's FFT: a cosine c cos(2pi(fy y/H + fx x/W))
    has two spectral lines |F| = c HW/2, so A^2 = c^2 HW/4 there and 0 elsewhere.  With
    every other line outside the 9x9 box, the box means at a line are A^2/w^2 and the
    minimum is the w = 9 one, A^2/81; s2 = sum c_i^2/2 (Parseval).  Hence each component
    is scaled by g_i = s2 / max(c_i^2 HW/324, s2): a strong line is attenuated, a weak
    one (box mean below s2) passes with gain exactly 1."""
    H, W = 64, 48
    c1, c2 = 1.0, 0.05
    K1, K2 = _cos(H, W, c1, 9, 13), _cos(H, W, c2, 25, 6)
    s2 = (c1 * c1 + c2 * c2) / 2
    g1 = s2 / max(c1 * c1 * H * W / 324, s2)
    g2 = s2 / max(c2 * c2 * H * W / 324, s2)
    assert g1 < 0.06 and g2 == 1.0
    out = oracle.wiener_dft(K1 + K2)
    assert np.max(np.abs(out - (g1 * K1 + g2 * K2))) < 1e-12


def test_wdft_closed_form_mirror_window_at_the_edge():
    """The mirror (e_N) extension of R-7 on the spectrum array: for a line in row 1
    (and its partner in row H-1) the 7- and 9-wide windows fold the line in twice,
    so the box means are A^2/9, A^2/25, 2A^2/49, 2A^2/81 and the minimum is 2A^2/81:
    gain = s2 / (2 A^2/81) = (c^2/2) / (c^2 HW/162) = 81/(HW)."""
    H, W = 40, 72
    K = _cos(H, W, 0.3, 1, 20)
    out = oracle.wiener_dft(K)
    assert np.max(np.abs(out - (81.0 / (H * W)) * K)) < 1e-12
