"""Pins for oracle a1 (SDA grouping + averaging)."""
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "denoise_counts.txt")
CONFIG_DEPTHS = (1, 2, 3, 4, 5, 10, 20, 25, 30, 50, 100, 300, 1200, 1800, 3600)


def _golden_counts():
    rows = []
    with open(GOLDEN) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                m, d, ns, cite = line.split()
                rows.append((int(m), int(d), int(ns), cite))
    return rows


@pytest.mark.parametrize("m,d,ns,cite", _golden_counts())
def test_denoise_count_law_paper(m, d, ns, cite):
    # the paper's printed SDA-frame counts
    assert oracle.sda_groups(m, d) == ns, cite


def test_grouping_edge_cases():
    assert oracle.sda_groups(10, 3) == 3      # S:193 floor semantics, 1 frame dropped
    assert oracle.sda_groups(10, 1) == 10
    assert oracle.sda_groups(5, 6) == -1      # S:189 DepthExceedsFrames
    assert oracle.sda_groups(5, 0) == -1


def _frames_with_sums(sums, d):
    """d uint8 frames (one pixel per sum) whose per-pixel sum is `sums`."""
    sums = np.asarray(sums, dtype=np.int64)
    fr = np.zeros((d, sums.size), dtype=np.uint8)
    q, r = sums // 255, sums % 255
    for j in range(d):
        fr[j] = np.where(j < q, 255, np.where(j == q, r, 0)).astype(np.uint8)
    return fr.reshape(d, 1, sums.size)


@pytest.mark.parametrize("d", CONFIG_DEPTHS)
def test_sda_mean_is_correctly_rounded_fp32(d):
    """The SDA mean equals the IEEE fp32 quotient fl32(s / d) of the exact
    integer sum (R-11).  numpy's float32 division is the independent
    correctly-rounded reference.  Exhaustive over every reachable sum for
    d <= 100, a 20k sample plus the extremes above."""
    smax = 255 * d
    if d <= 100:
        sums = np.arange(smax + 1)
    else:
        rng = np.random.default_rng(d)
        sums = np.unique(np.concatenate([rng.integers(0, smax + 1, 20000), [0, 1, smax - 1, smax]]))
    out = oracle.sda_average(_frames_with_sums(sums, d), d)[0, 0]
    ref = np.float32(sums.astype(np.float32)) / np.float32(d)
    assert out.dtype == np.float32
    np.testing.assert_array_equal(out.view(np.uint32), ref.astype(np.float32).view(np.uint32))


def test_rounding_formula_exhaustive_all_depths():
    """fl32(fl64(s)/d) == fl32(s)/fl32(d) for every s <= 255 d at every config depth
    (exact check of the double-rounding hazard the oracle's expression could have)."""
    for d in CONFIG_DEPTHS:
        s = np.arange(255 * d + 1, dtype=np.int64)
        a = (s.astype(np.float64) / d).astype(np.float32)
        b = s.astype(np.float32) / np.float32(d)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), d


def test_spec_examples():
    rng = np.random.default_rng(0)
    f = rng.integers(0, 256, (1, 7, 9), dtype=np.uint8)
    np.testing.assert_array_equal(oracle.sda_average(f, 1)[0], f[0].astype(np.float32))
    rep = np.repeat(f, 5, axis=0)
    np.testing.assert_array_equal(oracle.sda_average(rep, 5)[0], f[0].astype(np.float32))
    two = np.stack([np.zeros((4, 4), np.uint8), np.full((4, 4), 10, np.uint8)])
    np.testing.assert_array_equal(oracle.sda_average(two, 2)[0], np.full((4, 4), 5.0, np.float32))


def test_group_order_and_remainder():
    """Group i is frames [i d, (i+1) d); the remainder is dropped."""
    m, d = 11, 3
    f = np.arange(m, dtype=np.uint8)[:, None, None] * np.ones((1, 2, 2), np.uint8)
    out = oracle.sda_average(f, d)
    assert out.shape == (3, 2, 2)
    np.testing.assert_array_equal(out[:, 0, 0], np.array([1.0, 4.0, 7.0], np.float32))


@pytest.mark.parametrize("d", [2, 10, 30])
def test_averaging_noise_law(d):
    """Var(psi^SDA) = sigma_1^2 / d (S:243 within 20%).  Integer-rounded
    Gaussian noise has variance sigma^2 + 1/12."""
    rng = np.random.default_rng(d)
    sigma = 6.0
    trials = 30
    P = 4096
    ratios = []
    for _ in range(trials):
        fr = np.clip(np.rint(128 + sigma * rng.standard_normal((d, 1, P))), 0, 255).astype(np.uint8)
        v = oracle.sda_average(fr, d)[0].astype(np.float64).var()
        ratios.append(v / ((sigma ** 2 + 1.0 / 12.0) / d))
    assert abs(np.mean(ratios) - 1.0) < 0.2


# ---------------------------------------------------------------- f4: RGB -> luma
def test_luma_gray_is_identity():
    v = np.arange(256, dtype=np.uint8)
    rgb = np.stack([v, v, v])[None, :, None, :]          # planar [1,3,1,256]
    assert np.array_equal(oracle.rgb_to_luma(rgb, "planar", "fp32")[0, 0], v.astype(np.float32))
    assert np.array_equal(oracle.rgb_to_luma(rgb, "planar", "u8")[0, 0], v)


def test_luma_matches_fp64_formula_and_layouts():
    rng = np.random.default_rng(5)
    rgb = rng.integers(0, 256, size=(3, 3, 7, 9), dtype=np.uint8)
    y64 = 0.299 * rgb[:, 0].astype(np.float64) + 0.587 * rgb[:, 1] + 0.114 * rgb[:, 2]
    y = oracle.rgb_to_luma(rgb, "planar", "fp32")
    assert np.max(np.abs(y - y64)) <= 2 ** -24 * 256        # within fp32 rounding of the exact value
    inter = np.ascontiguousarray(np.moveaxis(rgb, 1, -1))
    assert np.array_equal(oracle.rgb_to_luma(inter, "interleaved", "fp32"), y)
    u = oracle.rgb_to_luma(rgb, "planar", "u8").astype(np.float64)
    assert np.max(np.abs(u - y64)) <= 0.5 + 1e-9


def test_luma_ties_round_half_to_even():
    # s = 299 R + 587 G + 114 B with s mod 1000 == 500 exactly
    ties = []
    for r in range(256):
        for g in range(0, 256, 5):
            for b in range(0, 256, 7):
                s = 299 * r + 587 * g + 114 * b
                if s % 1000 == 500:
                    ties.append((r, g, b, s // 1000))
    assert len(ties) > 10
    rgb = np.array([[t[0] for t in ties], [t[1] for t in ties], [t[2] for t in ties]], dtype=np.uint8)
    out = oracle.rgb_to_luma(rgb[None, :, None, :], "planar", "u8")[0, 0]
    expect = np.array([q + (q % 2) for (_, _, _, q) in ties], dtype=np.uint8)   # half to even
    assert np.array_equal(out, expect)
