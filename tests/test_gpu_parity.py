"""GPU <-> oracle parity through the C ABI (libprnu.so), on the same seeded inputs.

Tolerances (BASELINE.json north_star):
  SDA mean        bit-exact
  residual W      max |dW| <= 1e-3 intensity units
  fingerprint K   max |dK| * sqrt(sum_I2 / n_sda) <= 1e-3 intensity units (R-14)
  NCC             |d| <= 1e-5
  PCE             relative <= 1e-3 (tie rule R-19)
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

W_TOL = 1e-3
K_TOL = 1e-3
NCC_TOL = 1e-5
PCE_RTOL = 1e-3


@pytest.fixture(scope="module")
def prnu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1909_04573_b200 as m
    return m


def _rand_frames(m, H, W, seed, lo=0, hi=256):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return torch.randint(lo, hi, (m, H, W), generator=g, dtype=torch.uint8)


def _textured(b, H, W, seed):
    """fp32 planes with structure on every scale + noise, in [0, 255]."""
    g = np.random.default_rng(seed)
    y, x = np.mgrid[0:H, 0:W]
    out = []
    for i in range(b):
        f = 128 + 50 * np.sin(2 * np.pi * (x / g.uniform(5, 40) + y / g.uniform(5, 40)))
        f += 20 * np.cos(2 * np.pi * y / g.uniform(3, 9)) + g.normal(0, 4, (H, W))
        out.append(np.clip(f, 0, 255))
    return np.stack(out).astype(np.float32)


def k_metric(K_gpu, K_ref, den, n_sda):
    """R-14: error of the implied PRNU term K I in intensity units."""
    d = np.abs(K_gpu.astype(np.float64) - K_ref)
    return float((d * np.sqrt(den / n_sda)).max()), float(255 * d.max())


# ---------------------------------------------------------------- a1
@pytest.mark.parametrize("m,H,W,d", [(16, 64, 64, 4), (16, 64, 64, 1), (10, 33, 47, 3), (300, 17, 16, 300),
                                     (7, 5, 3, 2), (600, 24, 40, 257), (1, 1, 1, 1)])
def test_sda_average_bit_exact(prnu, m, H, W, d):
    fr = _rand_frames(m, H, W, m * 7 + d)
    got = prnu.sda_average(fr.cuda(), d).cpu().numpy()
    ref = oracle.sda_average(fr.numpy(), d)
    assert got.shape == ref.shape
    np.testing.assert_array_equal(got.view(np.uint32), ref.view(np.uint32))


def test_sda_average_extremes_bit_exact(prnu):
    """All-255 and alternating extremes at the largest config depth (3600)."""
    d = 3600
    fr = torch.full((d, 4, 16), 255, dtype=torch.uint8)
    fr[::2, :, ::3] = 0
    fr[::7, 1, :] = 1
    got = prnu.sda_average(fr.cuda(), d).cpu().numpy()
    np.testing.assert_array_equal(got.view(np.uint32), oracle.sda_average(fr.numpy(), d).view(np.uint32))


# ---------------------------------------------------------------- a2-a4
@pytest.mark.parametrize("b,H,W", [(1, 64, 64), (3, 37, 53), (2, 135, 240), (1, 16, 16), (2, 100, 333),
                                   (1, 270, 480),
                                   # strip staging: 16 <= H < 32 (mirrored rows, generic reflection),
                                   # H = 31/32/33 around the single-reflection threshold, wide and narrow
                                   (1, 17, 700), (2, 20, 333), (1, 31, 500), (1, 32, 257), (1, 33, 1000),
                                   (1, 300, 17)])
def test_residual_matches_oracle(prnu, b, H, W):
    I = _textured(b, H, W, H * W + b)
    got = prnu.residual(torch.from_numpy(I).cuda()).cpu().numpy()
    for i in range(b):
        ref = oracle.residual(I[i])
        err = np.abs(got[i] - ref).max()
        assert err <= W_TOL, (i, err)


@pytest.mark.parametrize("levels,windows,s0", [(1, (3,), 9.0), (2, (5, 9), 4.0), (3, (3, 5, 7, 9), 25.0),
                                               (5, (7,), 9.0), (6, (3, 9), 1.0)])
def test_residual_params_match_oracle(prnu, levels, windows, s0):
    I = _textured(1, 96, 130, levels)[0]
    p = prnu.DenoiseParams(sigma0_sq=s0, levels=levels, windows=windows)
    got = prnu.residual(torch.from_numpy(I).cuda(), p).cpu().numpy()
    ref = oracle.residual(I, sigma0_sq=s0, windows=windows, levels=levels)
    assert np.abs(got - ref).max() <= W_TOL


def test_residual_u8_and_zero_mean(prnu):
    fr = _rand_frames(2, 70, 90, 11, 30, 220)
    got = prnu.residual(fr.cuda(), zero_mean=True).cpu().numpy()
    for i in range(2):
        ref = oracle.residual(fr[i].numpy().astype(np.float32), zero_mean=True)
        assert np.abs(got[i] - ref).max() <= W_TOL
        assert np.abs(got[i].astype(np.float64).mean(axis=0)).max() < 1e-4
        assert np.abs(got[i].astype(np.float64).mean(axis=1)).max() < 1e-4


@pytest.mark.parametrize("H,W", [(17, 700), (31, 500), (33, 1000), (64, 64), (135, 241)])
def test_residual_u8_sizes(prnu, H, W):
    """u8 input (the level-1 u8 strip kernel) at heights around the staging thresholds."""
    fr = _rand_frames(2, H, W, H + W, 10, 245)
    got = prnu.residual(fr.cuda()).cpu().numpy()
    for i in range(2):
        assert np.abs(got[i] - oracle.residual(fr[i].numpy().astype(np.float32))).max() <= W_TOL


def test_residual_invariants(prnu):
    c = torch.full((2, 64, 96), 128.0, device="cuda")
    assert prnu.residual(c).abs().max().item() < 1e-4             # S:120 constant -> 0
    I = torch.from_numpy(np.round(_textured(1, 64, 96, 5))).cuda()
    d = prnu.residual(I + 10.0) - prnu.residual(I)               # S:130 offset invariance
    assert d.abs().max().item() < 1e-3
    with pytest.raises(prnu.PrnuError) as e:
        prnu.residual(torch.zeros((1, 15, 64), device="cuda"))
    assert e.value.code == 2


def test_residual_deterministic_and_batch_independent(prnu):
    I = torch.from_numpy(_textured(4, 80, 120, 9)).cuda()
    a = prnu.residual(I)
    b = prnu.residual(I)
    c = torch.cat([prnu.residual(I[i:i + 1]) for i in range(4)])
    assert torch.equal(a, b) and torch.equal(a, c)


# ---------------------------------------------------------------- a5-a6
def test_accumulate_finalize_match_oracle(prnu):
    H, W = 40, 56
    g = np.random.default_rng(0)
    Ws = g.normal(0, 2, (5, H, W)).astype(np.float32)
    Is = g.uniform(0, 255, (5, H, W)).astype(np.float32)
    Is[:, 0, 0] = 0.0   # eps floor
    num = torch.zeros((H, W), dtype=torch.float64, device="cuda")
    den = torch.zeros_like(num)
    prnu.fingerprint_accumulate(torch.from_numpy(Ws).cuda(), torch.from_numpy(Is).cuda(), num, den)
    rn, rd = np.zeros((H, W)), np.zeros((H, W))
    for i in range(5):
        oracle.mle_accumulate(Ws[i].astype(np.float64), Is[i], rn, rd)
    # fp32 inputs: products exact in fp64, same ascending order -> bit-identical
    assert np.array_equal(num.cpu().numpy(), rn) and np.array_equal(den.cpu().numpy(), rd)
    for zm in (False, True):
        K = prnu.fingerprint_finalize(num, den, zero_mean=zm).cpu().numpy()
        Kr = oracle.finalize(rn, rd, zero_mean=zm)
        assert np.abs(K - Kr).max() <= 1e-6 * max(1.0, np.abs(Kr).max())
    K = prnu.fingerprint_finalize(num, den).cpu().numpy().astype(np.float64)
    assert np.abs(K.mean(axis=0)).max() < 1e-6 and np.abs(K.mean(axis=1)).max() < 1e-6


@pytest.mark.parametrize("depth,batch", [(4, 1), (4, 3), (1, 16), (1, 5), (16, 1), (3, 2)])
def test_extract_config1_matches_oracle(prnu, depth, batch):
    """BASELINE config 1: 16 frames 64x64, d = 4 (and d = 1, 16, 3 with a dropped frame)."""
    v = synth.video("shift", 16, 64, 64, seed=0)
    fp = prnu.extract_fingerprint(v.frames.cuda(), depth, batch=batch)
    K, num, den, ns = oracle.extract_fingerprint(v.frames.numpy(), depth)
    assert fp.n_sda == ns == 16 // depth
    np.testing.assert_array_equal(fp.sum_I2.cpu().numpy(), den)     # DEN is exact on both sides
    prim, sec = k_metric(fp.K.cpu().numpy(), K, den, ns)
    assert prim <= K_TOL, (prim, sec)
    ncc_true = prnu.ncc(fp.K, v.K.cuda()).item()
    assert abs(ncc_true - oracle.ncc(K, v.K.numpy())) <= NCC_TOL
    assert ncc_true > 0.5 and abs(prnu.ncc(fp.K, v.K_other.cuda()).item()) < 0.1


def test_extract_depth1_bit_identical_to_conventional(prnu):
    """S:227 / S:241 / P:344: the d = 1 pipeline equals residual + accumulate + finalize."""
    v = synth.video("drift", 12, 72, 136, seed=4)
    fr = v.frames.cuda()
    fp = prnu.extract_fingerprint(fr, 1, batch=5)
    I = fr.float()
    Wr = prnu.residual(I)
    num = torch.zeros((72, 136), dtype=torch.float64, device="cuda")
    den = torch.zeros_like(num)
    prnu.fingerprint_accumulate(Wr, I, num, den)
    K = prnu.fingerprint_finalize(num, den)
    assert torch.equal(fp.sum_WI, num) and torch.equal(fp.sum_I2, den) and torch.equal(fp.K, K)


@pytest.mark.parametrize("H,W,d", [(1081, 1919, 1), (270, 481, 3), (33, 1000, 1)])
def test_extract_odd_sizes_bit_identical_to_conventional(prnu, H, W, d):
    """Odd widths (u8 rows not 16-byte aligned: no tensor map, thread-loaded staging)
    and odd heights: the fused extraction equals SDA + residual + accumulate +
    finalize bit for bit, and matches the oracle's K (R-14)."""
    m = 2 * d
    fr = _rand_frames(m, H, W, H + W + d, 20, 236).cuda()
    fp = prnu.extract_fingerprint(fr, d, batch=2)
    S = prnu.sda_average(fr, d)
    Wr = prnu.residual(S if d > 1 else fr)
    num = torch.zeros((H, W), dtype=torch.float64, device="cuda")
    den = torch.zeros_like(num)
    prnu.fingerprint_accumulate(Wr, S, num, den)
    assert torch.equal(fp.sum_I2, den)
    assert torch.equal(fp.sum_WI, num) and torch.equal(fp.K, prnu.fingerprint_finalize(num, den))
    if H * W <= 300_000:
        K_ref, _, den_ref, n = oracle.extract_fingerprint(fr.cpu().numpy(), d)
        assert k_metric(fp.K.cpu().numpy(), K_ref, den_ref, n)[0] <= K_TOL


@pytest.mark.parametrize("H,W,m,batch", [(64, 128, 10, 2), (33, 1024, 6, 3), (270, 480, 8, 4), (1080, 1920, 4, 2)])
def test_extract_depth2_pairs(prnu, H, W, m, batch):
    """d = 2 on TMA-stageable frames (W % 16 == 0, >= 32 rows): both frames of a group are
    staged by one depth-2 box in the analysis and the accumulation (S = (b0 + b1) / 2, R-11).
    Bit-identical to the u16-sum path (same frames at a base not 16-byte aligned) and to
    SDA average + residual + accumulate + finalize; K against the oracle (R-14); the
    extreme values 0 and 255 in both frames of a pair."""
    fr = _rand_frames(m, H, W, H + 7 * W + m, 0, 256).cuda()
    fr[0, :5] = 255
    fr[1, :5] = 255
    fr[0, 5:9] = 0
    fp = prnu.extract_fingerprint(fr, 2, batch=batch)
    raw = torch.empty(m * H * W + 16, dtype=torch.uint8, device="cuda")
    fr_u = raw[1:1 + m * H * W].view(m, H, W)   # misaligned base: the u16-sum path
    fr_u.copy_(fr)
    fu = prnu.extract_fingerprint(fr_u, 2, batch=batch)
    assert torch.equal(fp.sum_I2, fu.sum_I2) and torch.equal(fp.sum_WI, fu.sum_WI) and torch.equal(fp.K, fu.K)
    S = prnu.sda_average(fr, 2)
    Wr = prnu.residual(S)
    num = torch.zeros((H, W), dtype=torch.float64, device="cuda")
    den = torch.zeros_like(num)
    prnu.fingerprint_accumulate(Wr, S, num, den)
    assert torch.equal(fp.sum_I2, den) and torch.equal(fp.sum_WI, num)
    assert torch.equal(fp.K, prnu.fingerprint_finalize(num, den))
    if H * W <= 300_000:
        K_ref, _, den_ref, n = oracle.extract_fingerprint(fr.cpu().numpy(), 2)
        assert fp.n_sda == n == m // 2
        np.testing.assert_array_equal(fp.sum_I2.cpu().numpy(), den_ref)
        assert k_metric(fp.K.cpu().numpy(), K_ref, den_ref, n)[0] <= K_TOL


def test_extract_on_high_priority_stream_bit_identical(prnu):
    """The wave streams of an extraction inherit the caller stream's priority (their own
    context per priority); results do not depend on it."""
    v = synth.video("drift", 24, 64, 128, seed=3)
    fr = v.frames.cuda()
    ref = prnu.extract_fingerprint(fr, 1, batch=5)
    ref_K, ref_den = ref.K.clone(), ref.sum_I2.clone()
    hp = torch.cuda.Stream(priority=-1)
    hp.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(hp):
        fp = prnu.extract_fingerprint(fr, 1, batch=5)
    torch.cuda.current_stream().wait_stream(hp)
    assert torch.equal(fp.K, ref_K) and torch.equal(fp.sum_I2, ref_den)


def test_check_results_error_kinds(prnu):
    """SPEC's data-dependent error kinds (S:216 EmptyAccumulator, S:288 ConstantInput,
    S:297 DegenerateSurface) through the synchronous prnu_check_results; the asynchronous
    calls report them in-band (NaN / non-finite / zero)."""
    g = torch.Generator(device="cpu").manual_seed(5)
    a = torch.full((2, 32, 48), 3.0, device="cuda")             # zero variance
    b = torch.randn((2, 32, 48), generator=g).cuda()
    assert torch.isnan(prnu.ncc(a, b)).all()
    with pytest.raises(prnu.PrnuError) as e:
        prnu.ncc(a, b, check=True)
    assert e.value.code == 7
    prnu.ncc(b, b + 1.0, check=True)                            # a valid pair passes
    R = torch.randn((1, 64, 64), generator=g).cuda()
    res = prnu.pce(R, torch.zeros((1, 64, 64), device="cuda"))  # a constant (zero) surface
    assert (res.peak == 0).all()
    with pytest.raises(prnu.PrnuError) as e:
        prnu.pce(R, torch.zeros((1, 64, 64), device="cuda"), check=True)
    assert e.value.code == 8
    prnu.pce(R, R.clone(), check=True)
    with pytest.raises(prnu.PrnuError) as e:
        prnu.check_results(prnu.CHECK_SUM_I2, torch.zeros((64, 64), dtype=torch.float64, device="cuda"))
    assert e.value.code == 6
    fp = prnu.extract_fingerprint(synth.video("shift", 8, 64, 64, seed=1).frames.cuda(), 2, batch=2)
    prnu.check_results(prnu.CHECK_SUM_I2, fp.sum_I2)


def test_extract_deterministic_across_batches(prnu):
    v = synth.video("drift", 40, 64, 128, seed=2)
    fr = v.frames.cuda()
    ref = prnu.extract_fingerprint(fr, 2, batch=20).K.clone()
    for b in (1, 7, 20, 64):
        assert torch.equal(prnu.extract_fingerprint(fr, 2, batch=b).K, ref)


def test_extract_host_matches_device(prnu):
    v = synth.video("drift", 30, 64, 96, seed=8)
    dev = prnu.extract_fingerprint(v.frames.cuda(), 3, batch=4).K.cpu()
    ex = prnu.Extractor(64, 96, 3, batch=4, host=True)
    host = ex(v.frames.pin_memory()).K.clone()
    assert torch.equal(dev, host)


# ---------------------------------------------------------------- a7-a8
def test_ncc_matches_oracle(prnu):
    g = np.random.default_rng(3)
    a = g.normal(0.3, 1, (3, 123, 77)).astype(np.float32)
    b = (0.2 * a + g.normal(0, 1, a.shape)).astype(np.float32)
    got = prnu.ncc(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
    for i in range(3):
        assert abs(got[i] - oracle.ncc(a[i], b[i])) <= NCC_TOL
    x = torch.from_numpy(a[0]).cuda()
    assert abs(prnu.ncc(x, x).item() - 1) < 1e-12
    assert abs(prnu.ncc(x, -3 * x + 1).item() + 1) < 1e-12
    assert np.isnan(prnu.ncc(torch.ones_like(x), x).item())


def _pce_check(prnu, R, T, excl=5):
    res = prnu.pce(torch.from_numpy(R).cuda(), torch.from_numpy(T).cuda(), excl)
    res_al = prnu.pce(torch.from_numpy(R).cuda(), torch.from_numpy(T).cuda(), excl, aligned=True)
    for i in range(R.shape[0]):
        C = oracle.correlation_surface(R[i], T[i])
        p_al = oracle.match.pce_from_surface(C, excl, peak=(0, 0))[0]
        assert abs(res_al.pce[i].item() - p_al) <= PCE_RTOL * abs(p_al)
        gy, gx = res.peak_y[i].item(), res.peak_x[i].item()
        p_ref, peak_ref, v_ref = oracle.match.pce_from_surface(C, excl)
        if (gy, gx) != peak_ref:
            # R-19: only acceptable when the oracle's top two |C| nearly tie
            top = np.sort(np.abs(C).ravel())[-2:]
            assert (top[1] - top[0]) / top[1] < 1e-4, ((gy, gx), peak_ref)
            p_ref = oracle.match.pce_from_surface(C, excl, peak=(gy, gx))[0]
        assert abs(res.pce[i].item() - p_ref) <= PCE_RTOL * abs(p_ref)
        assert abs(res.peak[i].item() - C[gy, gx]) <= 1e-3 * np.abs(C).max()


def test_pce_matches_oracle_shifted(prnu):
    g = np.random.default_rng(5)
    T = g.normal(0, 1, (3, 96, 160)).astype(np.float32)
    R = np.stack([np.roll(T[i], (i * 7, i * 13 + 1), axis=(0, 1)) + g.normal(0, 3, T[i].shape)
                  for i in range(3)]).astype(np.float32)
    _pce_check(prnu, R, T)
    res = prnu.pce(torch.from_numpy(R).cuda(), torch.from_numpy(T).cuda())
    assert [(res.peak_y[i].item(), res.peak_x[i].item()) for i in range(3)] == [(0, 1), (7, 14), (14, 27)]


def test_pce_matches_oracle_null(prnu):
    g = np.random.default_rng(6)
    R = g.normal(0, 1, (4, 64, 80)).astype(np.float32)
    T = g.normal(0, 1, (4, 64, 80)).astype(np.float32)
    _pce_check(prnu, R, T)
    _pce_check(prnu, R[:1, :10, :9].copy(), T[:1, :10, :9].copy(), excl=5)   # neighbourhood wraps


def test_camera_identification_small(prnu):
    """Config-4 shape at small scale: 4 cameras, K_hat (.) I_q templates, PCE matrix;
    diagonal > 60 > off-diagonal (directional) and parity of every entry."""
    H, W, n = 128, 192, 4
    fps, queries, qres = [], [], []
    for c in range(n):
        v = synth.video("drift", 61, H, W, seed=1, camera=c, sigma_n=2.0)
        fps.append(prnu.extract_fingerprint(v.frames[:60].cuda(), 6).K)
        queries.append(v.frames[60])
    Iq = torch.stack(queries).cuda()
    Rq = prnu.residual(Iq, zero_mean=True)
    M = np.zeros((n, n))
    for c in range(n):
        T = prnu.pce_template(fps[c], Iq)
        res = prnu.pce(Rq, T)
        M[:, c] = res.pce.cpu().numpy()
        for q in range(n):
            Rr = oracle.residual(queries[q].numpy().astype(np.float32), zero_mean=True)
            Tr = oracle.pce_template(fps[c].cpu().numpy(), queries[q].numpy())
            ref = oracle.pce(Rr, Tr)[0]
            assert abs(M[q, c] - ref) <= PCE_RTOL * abs(ref) + 1e-6
    assert np.all(np.diag(M) > 60)
    assert np.all(M[~np.eye(n, dtype=bool)] < 60)
    # f4 H0/H1 harness on the same matrix: perfect separation at the paper's threshold
    rates = prnu.detection_rates(M)
    assert rates["tpr"] == 1.0 and rates["fpr"] == 0.0 and rates["n_h0"] == n * (n - 1)
    assert prnu.roc(np.diag(M), M[~np.eye(n, dtype=bool)])[2] == 1.0


def test_launch_counter_advances(prnu):
    before = prnu.kernel_launches()
    prnu.residual(torch.zeros((1, 64, 64), device="cuda"))
    n = prnu.kernel_launches() - before
    # 4 synthesis launches; per analysis level 1 launch (fused) or 2 (DWT + shrink, split levels)
    assert 8 <= n <= 12, n


# ---------------------------------------------------------------- f1 block-wise
@pytest.mark.parametrize("H,W,block", [(130, 170, 50), (512, 1024, 500), (96, 64, 32)])
def test_block_match_matches_oracle(prnu, H, W, block):
    """per-tile aligned PCE and NCC, edge tiles kept."""
    g = np.random.default_rng(H + W)
    T = g.normal(0, 1, (H, W)).astype(np.float32)
    R = (0.2 * T + g.normal(0, 1, (H, W))).astype(np.float32)
    plan = prnu.BlockPlan(H, W, block)
    pce, ncc = plan(torch.from_numpy(R).cuda(), torch.from_numpy(T).cuda())
    ref = oracle.blockwise_match(R, T, block)
    assert plan.n_tiles == len(ref) and plan.tiles() == [r[:4] for r in ref]
    pce, ncc = pce.cpu().numpy(), ncc.cpu().numpy()
    for i, (y, x, h, w, p, c) in enumerate(ref):
        assert abs(pce[i] - p) <= PCE_RTOL * abs(p), (i, pce[i], p)
        assert abs(ncc[i] - c) <= NCC_TOL


def test_block_match_fhd_directional(prnu):
    """Full-HD query vs its camera's fingerprint, 500x500 blocks (12 tiles incl.
    80-row and 420-column edge tiles): matched blocks exceed the threshold."""
    v = synth.video("drift", 201, 1080, 1920, seed=6, sigma_n=2.0, device="cuda")
    fp = prnu.extract_fingerprint(v.frames[:200], 10, batch=20)
    q = v.frames[200:201]
    R = prnu.residual(q, zero_mean=True)[0]
    T = prnu.pce_template(fp.K, q)[0]
    pce, ncc = prnu.block_match(R, T, 500)
    assert pce.numel() == 12
    full = [i for i, (y, x, h, w) in enumerate(prnu.BlockPlan(1080, 1920, 500).tiles()) if h == 500 and w == 500]
    assert (pce[full] > 60).all()
    ref = oracle.blockwise_match(R.cpu().numpy(), T.cpu().numpy(), 500)
    for i, r in enumerate(ref):
        assert abs(pce[i].item() - r[4]) <= PCE_RTOL * abs(r[4])
        assert abs(ncc[i].item() - r[5]) <= NCC_TOL


# ---------------------------------------------------------------- f4 stride (I-frame) emulation
@pytest.mark.parametrize("stride,batch", [(3, 2), (1, 16), (5, 64), (16, 4)])
def test_stride_extraction_equals_selected_frames(prnu, stride, batch):
    """S:224 stride(k): keep frames with index = 0 mod k, then conventional; bit-identical
    to extracting the explicitly selected frames, and matching the oracle."""
    v = synth.video("shift", 16, 64, 64, seed=3)
    fr = v.frames.cuda()
    fs = prnu.extract_fingerprint_stride(fr, stride, batch=batch)
    sel = fr[::stride].contiguous()
    assert fs.n_sda == sel.shape[0] == -(-16 // stride)
    ref = prnu.extract_fingerprint(sel, 1, batch=batch)
    assert torch.equal(fs.K, ref.K) and torch.equal(fs.sum_WI, ref.sum_WI)
    K, num, den, ns = oracle.extract_fingerprint(sel.cpu().numpy(), 1)
    assert k_metric(fs.K.cpu().numpy(), K, den, ns)[0] <= K_TOL


def test_stride_vs_sda_directional(prnu):
    """S:229/S:610 (Fig. 6 direction): with equal denoise counts, SDA-30
    estimates K better than stride-30 (I-FE emulation)."""
    v = synth.video("drift", 600, 180, 320, seed=2, device="cuda")
    f_sda = prnu.extract_fingerprint(v.frames, 30, batch=20)
    f_str = prnu.extract_fingerprint_stride(v.frames, 30, batch=20)
    assert f_sda.n_sda == f_str.n_sda == 20
    assert prnu.ncc(f_sda.K, v.K).item() > prnu.ncc(f_str.K, v.K).item() + 0.05


def test_multi_depth_one_upload_matches_device(prnu):
    """prnu_extract_multi_host: one chunked upload, several depths; each fingerprint
    bit-identical to the device-frame extraction (waves straddle upload chunks)."""
    v = synth.video("drift", 300, 72, 96, seed=11)
    host = v.frames.pin_memory()
    depths = [1, 50, 7, 300]
    mx = prnu.MultiExtractor(300, 72, 96, depths, batch=16)
    K = mx(host).clone()
    assert mx.n_sda == [300, 6, 42, 1]
    for i, d in enumerate(depths):
        ref = prnu.extract_fingerprint(v.frames.cuda(), d, batch=16)
        assert torch.equal(K[i], ref.K.cpu()), d
        assert torch.equal(mx.sums[i, 1], ref.sum_I2)


# ---------------------------------------------------------------- f4 luma
@pytest.mark.gpu
@pytest.mark.parametrize("layout", ["planar", "interleaved"])
@pytest.mark.parametrize("n,H,W", [(1, 4, 4), (3, 37, 52), (2, 270, 480)])
def test_rgb_to_luma_bit_exact(prnu, layout, n, H, W):
    g = torch.Generator().manual_seed(11 + H)
    shape = (n, 3, H, W) if layout == "planar" else (n, H, W, 3)
    rgb = torch.randint(0, 256, shape, generator=g, dtype=torch.uint8)
    rgb[0].view(-1)[:8] = 255
    rgb[-1].view(-1)[-8:] = 0
    for dt, rnd in ((torch.float32, "fp32"), (torch.uint8, "u8")):
        y = prnu.rgb_to_luma(rgb.cuda(), layout, dt).cpu().numpy()
        ref = oracle.rgb_to_luma(rgb.numpy(), layout, rnd)
        assert y.dtype == ref.dtype and np.array_equal(y.view(np.uint8), ref.view(np.uint8))


@pytest.mark.gpu
def test_rgb_to_luma_errors(prnu):
    with pytest.raises(prnu.PrnuError):
        prnu.rgb_to_luma(torch.zeros((1, 3, 3, 3), dtype=torch.uint8, device="cuda"))   # H*W not a multiple of 4


# ---------------------------------------------------------------- f2 WDFT (R-23)
@pytest.mark.gpu
@pytest.mark.parametrize("B,H,W", [(1, 16, 24), (2, 130, 170), (1, 270, 480)])
def test_wdft_matches_oracle(prnu, B, H, W):
    rng = np.random.default_rng(H * W)
    y, x = np.mgrid[0:H, 0:W]
    Ks = []
    for b in range(B):
        K = rng.normal(0, 0.01, (H, W)) + 0.03 * np.cos(2 * np.pi * (3 * y / H + 7 * x / W + 0.3 * b))
        Ks.append((K - K.mean()).astype(np.float32))
    Kt = torch.from_numpy(np.stack(Ks)).cuda()
    out = prnu.WdftPlan(H, W, B)(Kt).cpu().numpy()
    for b in range(B):
        ref = oracle.wiener_dft(Ks[b].astype(np.float64))
        err = np.max(np.abs(out[b] - ref)) / np.max(np.abs(Ks[b]))
        assert err <= 1e-4, err


@pytest.mark.gpu
def test_wdft_closed_form_gpu(prnu):
    """The GPU path against R-23's closed form (tests/test_oracle_match.py): an isolated
    strong line is scaled by s2/(c1^2 HW/324), a weak one passes with gain 1, and a line
    in spectrum row 1 (mirror window folds it in twice) is scaled by 81/(HW)."""
    def cos(H, W, c, fy, fx):
        y, x = np.mgrid[0:H, 0:W]
        return c * np.cos(2 * np.pi * (fy * y / H + fx * x / W))
    H, W = 64, 48
    K1, K2 = cos(H, W, 1.0, 9, 13), cos(H, W, 0.05, 25, 6)
    s2 = (1.0 + 0.05 ** 2) / 2
    want_a = (s2 / (H * W / 324)) * K1 + K2
    H2, W2 = 40, 72
    K3 = cos(H2, W2, 0.3, 1, 20)
    want_b = (81.0 / (H2 * W2)) * K3
    for K, want in ((K1 + K2, want_a), (K3, want_b)):
        got = prnu.wdft(torch.from_numpy(K.astype(np.float32)).cuda()).cpu().numpy()
        assert np.max(np.abs(got - want)) <= 1e-5 * np.max(np.abs(K)), np.max(np.abs(got - want))


@pytest.mark.gpu
def test_wdft_fingerprint_fhd(prnu):
    """On a real (synthetic-camera) fingerprint at FHD: parity and it keeps the PRNU
    (NCC with the true K does not drop)."""
    v = synth.video("drift", 100, 1080, 1920, seed=3)
    fp = prnu.extract_fingerprint(v.frames.cuda(), 50, batch=2)
    Kw = prnu.wdft(fp.K)
    ref = oracle.wiener_dft(fp.K.cpu().numpy().astype(np.float64))
    err = np.max(np.abs(Kw.cpu().numpy() - ref)) / float(fp.K.abs().max())
    assert err <= 1e-4, err
    assert prnu.ncc(Kw, v.K.cuda()).item() >= prnu.ncc(fp.K, v.K.cuda()).item() - 0.02


@pytest.mark.parametrize("m,H,W,d", [(16, 64, 64, 4), (40, 135, 240, 1), (60, 96, 130, 20)])
def test_graph_extractor_bit_identical(prnu, m, H, W, d):
    """The CUDA-graph-captured extraction (GraphExtractor) replays to the same bits as the
    eager Extractor, across replays and after the static input buffer is rewritten."""
    fr = _rand_frames(m, H, W, 3 + d)
    ex = prnu.Extractor(H, W, d, 8)
    gx = prnu.GraphExtractor(m, H, W, d, 8)
    a = ex(fr.cuda())
    b = gx(fr.cuda())
    assert torch.equal(a.K, b.K) and torch.equal(a.sum_WI, b.sum_WI) and torch.equal(a.sum_I2, b.sum_I2)
    fr2 = _rand_frames(m, H, W, 99 + d)
    a2 = ex(fr2.cuda()).K.clone()
    assert torch.equal(gx(fr2.cuda()).K, a2) and torch.equal(gx().K, a2)


def test_pce_cached_residual_spectrum_bit_identical(prnu):
    """prnu_pce_residual_spectrum + prnu_pce_cached (one FFT of the residuals for many
    template batches) gives the bits of prnu_pce for every template batch."""
    H, W, b = 96, 130, 3
    R = torch.from_numpy(_textured(b, H, W, 5) - 128.0).cuda()
    Ts = [torch.from_numpy(_textured(b, H, W, 10 + k) - 128.0).cuda() for k in range(3)]
    plan = prnu.PcePlan(H, W, b)
    ref = [plan(R, T) for T in Ts]
    plan.set_residual(R)
    for T, r in zip(Ts, ref):
        got = plan.match(T)
        assert torch.equal(got.pce, r.pce) and torch.equal(got.peak_y, r.peak_y) and torch.equal(got.peak, r.peak)


@pytest.mark.parametrize("H,W", [(720, 1280), (96, 160), (45, 62), (27, 53)])
def test_pce_cached_template_bit_identical(prnu, H, W):
    """prnu_pce_cached_template (the template K (.) Iq formed inside the row transform,
    or staged on the cuFFT paths) gives the bits of prnu_pce_cached(prnu_pce_template);
    both agree with the oracle.  Sizes: fused rows + columns, cuFFT rows + columns,
    2-D cuFFT (odd W)."""
    b = 2
    g = np.random.default_rng(H + W)
    I = torch.from_numpy(g.integers(0, 256, (b, H, W), dtype=np.uint8)).cuda()
    K = torch.from_numpy(g.normal(0, 0.02, (H, W)).astype(np.float32)).cuda()
    R = prnu.residual(I, zero_mean=True)
    plan = prnu.PcePlan(H, W, b)
    plan.set_residual(R)
    ref = plan.match(prnu.pce_template(K, I))
    got = plan.match_template(K, I)
    assert torch.equal(got.pce, ref.pce) and torch.equal(got.peak_y, ref.peak_y) and torch.equal(got.peak, ref.peak)
    if H * W <= 96 * 160:
        for i in range(b):
            Tn = oracle.pce_template(K.cpu().numpy(), I[i].cpu().numpy())
            p_ref = oracle.pce(R[i].cpu().numpy().astype(np.float64), Tn)[0]
            assert abs(got.pce[i].item() - p_ref) <= PCE_RTOL * abs(p_ref) + 1e-6


def test_pce_matrix_matches_single_plan(prnu):
    """PceMatrix (plans dealt over streams) gives, row by row, the bits of one plan's
    match_template for each fingerprint."""
    H, W, b, n = 96, 160, 3, 5
    g = np.random.default_rng(11)
    I = torch.from_numpy(g.integers(0, 256, (b, H, W), dtype=np.uint8)).cuda()
    Ks = torch.from_numpy(g.normal(0, 0.02, (n, H, W)).astype(np.float32)).cuda()
    R = prnu.residual(I, zero_mean=True)
    pm = prnu.PceMatrix(H, W, b, streams=3)
    pm.set_queries(R, I)
    got = pm(Ks)
    plan = prnu.PcePlan(H, W, b)
    plan.set_residual(R)
    for c in range(n):
        ref = plan.match_template(Ks[c], I)
        assert torch.equal(got.pce[c], ref.pce) and torch.equal(got.peak_y[c], ref.peak_y)
        assert torch.equal(got.peak[c], ref.peak)


def test_camera_batch_extractor_matches_single(prnu):
    """Cameras dealt over several streams give each camera's single-stream fingerprint."""
    vids = [_rand_frames(20, 64, 96, 40 + c).cuda() for c in range(5)]
    K = prnu.CameraBatchExtractor(64, 96, 4, 3, streams=3)(vids)
    for c in range(5):
        assert torch.equal(K[c], prnu.extract_fingerprint(vids[c], 4, batch=3).K)


def test_residual_random_shapes(prnu):
    """24 seeded random plane shapes (16..420 x 16..700), levels 1..4, u8 and fp32
    input: every output against the oracle (catches staging/segment/strip edge cases)."""
    g = np.random.default_rng(2024)
    for case in range(24):
        H, W = int(g.integers(16, 421)), int(g.integers(16, 701))
        lv = int(g.integers(1, 5))
        while H < (1 << lv) or W < (1 << lv):
            lv -= 1
        p = prnu.DenoiseParams(levels=lv)
        fr = torch.from_numpy(g.integers(0, 256, (2, H, W), dtype=np.uint8))
        src = fr.cuda() if case % 2 == 0 else fr.float().cuda()
        got = prnu.residual(src, p).cpu().numpy()
        for i in range(2):
            ref = oracle.residual(fr[i].numpy().astype(np.float32), levels=lv)
            err = np.abs(got[i] - ref).max()
            assert err <= W_TOL, (case, H, W, lv, i, err)


def test_extract_random_configs(prnu):
    """10 seeded random extraction configurations (size, frame count, depth, batch):
    K against the oracle (R-14), n_sda = floor(m/d), sum_I2 bit-exact."""
    g = np.random.default_rng(77)
    for case in range(10):
        H, W = int(g.integers(16, 201)), int(g.integers(16, 241))
        m = int(g.integers(2, 41))
        d = int(g.integers(1, m + 1))
        batch = int(g.integers(1, 17))
        fr = torch.from_numpy(g.integers(10, 246, (m, H, W), dtype=np.uint8))
        fp = prnu.extract_fingerprint(fr.cuda(), d, batch=batch)
        K_ref, _, den, n = oracle.extract_fingerprint(fr.numpy(), d)
        assert fp.n_sda == n == m // d, (case, m, d)
        np.testing.assert_array_equal(fp.sum_I2.cpu().numpy(), den)
        assert k_metric(fp.K.cpu().numpy(), K_ref, den, n)[0] <= K_TOL, (case, H, W, m, d, batch)


@pytest.mark.parametrize("H,W", [(100, 256), (100, 336), (120, 512), (70, 400)])
def test_residual_short_deep_levels(prnu, H, W):
    """Deep levels with 16..31 input rows (level 4 of H = 100: 18 rows), where a block's
    mirrored rows can wrap through both plane edges: thread-staged, all outputs vs the oracle."""
    I = _textured(2, H, W, H + 3 * W)
    for src in (torch.from_numpy(I).cuda(), torch.from_numpy(np.round(I).astype(np.uint8)).cuda()):
        got = prnu.residual(src).cpu().numpy()
        for i in range(2):
            ref = oracle.residual(src[i].cpu().numpy().astype(np.float32))
            assert np.abs(got[i] - ref).max() <= W_TOL


@pytest.mark.parametrize("B,H,W,kb", [(3, 720, 1280, 1), (2, 45, 62, 2), (2, 7, 9, 1)])
def test_pce_template_bit_exact(prnu, B, H, W, kb):
    """S:305 / R-18: T = K (.) (float)Iq, one fp32 product per pixel: bit-exact against
    numpy for the 4-pixel vector path (P % 4 == 0) and the scalar path (odd P)."""
    g = np.random.default_rng(H + W)
    K = g.normal(0, 0.01, (kb, H, W)).astype(np.float32)
    I = g.integers(0, 256, (B, H, W), dtype=np.uint8)
    got = prnu.pce_template(torch.from_numpy(K[0] if kb == 1 else K).cuda(), torch.from_numpy(I).cuda()).cpu().numpy()
    want = (K if kb > 1 else K[[0] * B]) * I.astype(np.float32)
    assert got.shape == (B, H, W) and np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("H,W", [(45, 60), (27, 54), (125, 250), (64, 2), (2, 16), (48, 40), (48, 54), (45, 62),
                                 (720, 1280), (64, 6), (27, 4)])
def test_pce_fft235_sizes_match_oracle(prnu, H, W):
    """PCE at plane sizes whose factors are 3 and 5 only, powers of two, and tiny / flat
    planes, against the oracle's FFT-based surface (R-17, R-19): shifted, null and
    affine pairs."""
    g = np.random.default_rng(H * 7 + W)
    T = g.normal(0, 1, (3, H, W)).astype(np.float32)
    R = np.stack([np.roll(T[0], (1, 3 % W), axis=(0, 1)) + g.normal(0, 0.5, (H, W)),
                  g.normal(0, 1, (H, W)), T[2] * 2.0 + 1.0]).astype(np.float32)
    _pce_check(prnu, R, T, excl=min(5, (min(H, W) - 1) // 2))
