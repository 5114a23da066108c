"""Pins for the oracle's MLE accumulation (a5), finalize + zero-mean (a6) and the
composed fingerprint path: Eq. (2) P:151-155."""
import numpy as np
import pytest
import torch

import oracle
import synth


def test_accumulate_spec_example():
    """empty acc + (W = 2, I = 3) -> sum_WI = 6, sum_I2 = 9."""
    num = np.zeros((3, 4))
    den = np.zeros((3, 4))
    oracle.mle_accumulate(np.full((3, 4), 2.0), np.full((3, 4), 3.0, np.float32), num, den)
    assert np.all(num == 6.0) and np.all(den == 9.0)
    # khat = 2/3 before zero-mean, 0 after
    np.testing.assert_allclose(oracle.finalize(num, den, zero_mean=False), 2.0 / 3.0, rtol=1e-15)
    assert np.abs(oracle.finalize(num, den, zero_mean=True)).max() < 1e-15
    # S:210 additivity
    oracle.mle_accumulate(np.full((3, 4), 2.0), np.full((3, 4), 3.0, np.float32), num, den)
    assert np.all(num == 12.0) and np.all(den == 18.0)


def test_eps_floor():
    """sum_I2 = 0 at a pixel -> finite khat (eps floor)."""
    num = np.zeros((2, 2))
    den = np.ones((2, 2))
    den[0, 0] = 0.0
    K = oracle.finalize(num, den, zero_mean=False)
    assert np.all(np.isfinite(K))


def test_mle_recovers_K_exactly():
    """Closed form: if W_i = K (.) I_i exactly then K_hat (pre-ZM) = K."""
    rng = np.random.default_rng(0)
    K = rng.normal(0, 0.02, (16, 24))
    num, den = np.zeros_like(K), np.zeros_like(K)
    for i in range(5):
        I = rng.uniform(20, 230, K.shape).astype(np.float32)
        oracle.mle_accumulate(K * I.astype(np.float64), I, num, den)
    np.testing.assert_allclose(oracle.finalize(num, den, zero_mean=False), K, rtol=1e-13, atol=1e-16)


def test_zero_mean_properties():
    """S:135-140 rows then columns; equals the closed form x - r_i - c_j + t,
    leaves every row and column mean at 0, and is idempotent."""
    rng = np.random.default_rng(1)
    x = rng.normal(3, 2, (11, 17))
    z = oracle.zero_mean(x)
    closed = x - x.mean(axis=1, keepdims=True) - x.mean(axis=0, keepdims=True) + x.mean()
    np.testing.assert_allclose(z, closed, atol=1e-13)
    assert np.abs(z.mean(axis=0)).max() < 1e-14
    assert np.abs(z.mean(axis=1)).max() < 1e-14
    np.testing.assert_allclose(oracle.zero_mean(z), z, atol=1e-14)
    assert np.abs(oracle.zero_mean(np.full((4, 5), 5.0))).max() == 0.0


def test_depth1_equals_conventional_composition():
    """S:227/S:241 (and P:344 "SDA-1 is the same as conventional"): the d = 1
    path equals residual + accumulate + finalize on the widened u8 frames, bit-exact."""
    v = synth.video("shift", 6, 32, 40, seed=3)
    fr = v.frames.numpy()
    K, num, den, ns = oracle.extract_fingerprint(fr, 1)
    assert ns == 6
    n2, d2 = np.zeros((32, 40)), np.zeros((32, 40))
    for i in range(6):
        I = fr[i].astype(np.float32)
        oracle.mle_accumulate(oracle.residual(I), I, n2, d2)
    assert np.array_equal(num, n2) and np.array_equal(den, d2)
    assert np.array_equal(K, oracle.finalize(n2, d2))


def test_config1_directional():
    """BASELINE config 1 (16 frames 64x64, d = 4): the fingerprint correlates with
    the true K and not with another camera's K (directional, not parity)."""
    v = synth.video("shift", 16, 64, 64, seed=0)
    Kt, Ko = v.K.double().numpy(), v.K_other.double().numpy()
    for d in (4, 1):
        K, _, _, ns = oracle.extract_fingerprint(v.frames.numpy(), d)
        assert ns == 16 // d
        assert oracle.ncc(K, Kt) > 0.5
        assert abs(oracle.ncc(K, Ko)) < 0.1


def test_synth_is_deterministic():
    a = synth.video("drift", 3, 24, 40, seed=5).frames
    b = synth.video("drift", 3, 24, 40, seed=5).frames
    assert torch.equal(a, b)


def _groups_by_hand(fr, d):
    """SDA frames of the disjoint groups [i d, (i+1) d), i < floor(m/d) (P:124,
    P:170-175), written out with numpy: the exact integer sum of the
    group's frames over d, rounded once to fp32 (R-11; test_oracle_sda pins this
    rounding against IEEE fp32 division)."""
    m = fr.shape[0]
    out = []
    for i in range(m // d):
        s = fr[i * d:(i + 1) * d].astype(np.int64).sum(axis=0)
        out.append((s.astype(np.float64) / d).astype(np.float32))
    return out


@pytest.mark.parametrize("m,d", [(11, 3), (16, 4), (9, 2), (7, 7), (5, 1)])
def test_extract_fingerprint_groups_pinned(m, d):
    """oracle_extract_fingerprint at depth d > 1 with a remainder (m mod d frames
    dropped) equals, bit for bit, an explicit loop over the disjoint groups
    [i d, (i+1) d): hand-computed SDA frame -> residual -> MLE accumulate in
    ascending i -> finalize.  A wrong group stride
    (overlapping or shifted groups), a wrong group count or the remainder frames
    leaking in would change the sums."""
    v = synth.video("shift", m, 24, 40, seed=7)
    fr = v.frames.numpy()
    K, num, den, ns = oracle.extract_fingerprint(fr, d)
    assert ns == m // d
    n2, d2 = np.zeros((24, 40)), np.zeros((24, 40))
    for S in _groups_by_hand(fr, d):
        oracle.mle_accumulate(oracle.residual(S), S, n2, d2)
    assert np.array_equal(num, n2) and np.array_equal(den, d2)
    assert np.array_equal(K, oracle.finalize(n2, d2))
    # the m mod d remainder does not enter: overwrite it, same result
    if m % d:
        fr2 = fr.copy()
        fr2[ns * d:] = 255 - fr2[ns * d:]
        K2, num2, den2, _ = oracle.extract_fingerprint(fr2, d)
        assert np.array_equal(num2, num) and np.array_equal(den2, den)
    # every frame of every group does enter: perturb the last frame of the last group
    fr3 = fr.copy()
    fr3[ns * d - 1] ^= 1
    _, _, den3, _ = oracle.extract_fingerprint(fr3, d)
    assert not np.array_equal(den3, den)


def test_extract_fingerprint_overlap_detected():
    """The pin above distinguishes disjoint from overlapping groups: groups of the
    same depth at stride 1 give different sums (so the equality is not vacuous)."""
    v = synth.video("shift", 8, 24, 40, seed=8)
    fr = v.frames.numpy()
    _, num, den, _ = oracle.extract_fingerprint(fr, 4)
    n2, d2 = np.zeros((24, 40)), np.zeros((24, 40))
    for i in range(2):   # overlapping: frames [i, i + 4)
        S = (fr[i:i + 4].astype(np.int64).sum(0) / 4.0).astype(np.float32)
        oracle.mle_accumulate(oracle.residual(S), S, n2, d2)
    assert not np.array_equal(den, d2)


def test_extract_fingerprint_chunked_matches():
    """oracle.parallel.extract_fingerprint_chunked (partial sums of contiguous runs
    of groups in worker processes, added in order) equals the sequential oracle up
    to the regrouping of fp64 additions."""
    from oracle import parallel
    v = synth.video("shift", 23, 32, 48, seed=9)
    fr = v.frames.numpy()
    for d in (1, 3):
        K, num, den, ns = oracle.extract_fingerprint(fr, d)
        K2, num2, den2, ns2 = parallel.extract_fingerprint_chunked(fr, d, workers=2, chunks=3)
        assert ns2 == ns
        np.testing.assert_allclose(num2, num, rtol=1e-13, atol=1e-12)
        np.testing.assert_allclose(den2, den, rtol=1e-14)
        np.testing.assert_allclose(K2, K, rtol=1e-10, atol=1e-14)


def test_oracle_pool_matches_direct_calls():
    """oracle.parallel.OraclePool (worker processes + shared memory) returns what the
    oracle returns when called directly."""
    from oracle import parallel
    v = synth.video("shift", 8, 24, 32, seed=12)
    fr = v.frames.numpy()
    with parallel.OraclePool(workers=2) as pool:
        f = pool.fingerprint(fr, 4)
        r = pool.residual(fr[0])
        K, _, den, ns = oracle.extract_fingerprint(fr, 4)
        Kp, denp, nsp = f.get()
        assert nsp == ns and np.array_equal(Kp, K) and np.array_equal(denp, den)
        R = oracle.residual(fr[0].astype(np.float32), zero_mean=True)
        assert np.array_equal(r.get(), R)
        T = oracle.pce_template(K, fr[1])
        p, peak, gap, _ = pool.pce(R, T).get()
        p_ref, peak_ref, _ = oracle.pce(R, T)
        assert p == p_ref and peak == peak_ref
