"""Full-size parity (BASELINE.json configs 2-5) through the C ABI, in the launch
configuration bench.py times (waves of 360 frames, three streams), against the fp64 oracle on
outputs it can compute in seconds, plus properties that hold at any size.

Tolerances as in test_gpu_parity.py."""
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
BENCH_BATCH = 360   # bench.py default for 1800 frames: 5 equal waves


@pytest.fixture(scope="module")
def prnu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1909_04573_b200 as m
    return m


def k_metric(K_gpu, K_ref, den, n_sda):
    d = np.abs(K_gpu.astype(np.float64) - K_ref)
    return float((d * np.sqrt(den / n_sda)).max())


@pytest.fixture(scope="module")
def video_c2():
    """Config 2: 1800 (+1 query) frames 1920x1080, the drift recipe."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    v = synth.video("drift", 1801, 1080, 1920, seed=0, device="cuda")
    return v


def test_c2_depth50_full_oracle(prnu, video_c2, parity_report):
    """Config 2, SDA depth 50: the whole 36-frame fingerprint against the oracle."""
    fr = video_c2.frames[:1800]
    fp = prnu.extract_fingerprint(fr, 50, batch=36)
    K_ref, num, den, ns = oracle.extract_fingerprint(fr.cpu().numpy(), 50)
    assert fp.n_sda == ns == 36
    np.testing.assert_array_equal(fp.sum_I2.cpu().numpy(), den)      # exact: same fp32 SDA frames, same order
    Kg = fp.K.cpu().numpy()
    prim = k_metric(Kg, K_ref, den, ns)
    rho = prnu.ncc(fp.K, video_c2.K).item()
    d_ncc = abs(rho - oracle.ncc(K_ref, video_c2.K.cpu().numpy()))
    parity_report(f"C2 d=50: R-14 primary {prim:.3e}, secondary 255*max|dK| "
          f"{255.0 * float(np.abs(Kg.astype(np.float64) - K_ref).max()):.3e}, |dNCC| {d_ncc:.2e}")
    assert prim <= K_TOL
    assert d_ncc <= NCC_TOL
    assert rho > 0.9


def test_c2_depth1_full_oracle(prnu, video_c2, parity_report):
    """Config 2, conventional (1800 denoisings), in the bench configuration (waves
    of 360 frames over the library's three streams): the WHOLE 1800-frame
    fingerprint against the oracle ("SDA-1 is the same as conventional",
    P:413).  The oracle's fingerprint is computed by worker processes on every
    host core (oracle.parallel.extract_fingerprint_chunked: partial sums of
    contiguous frame runs, added in order; ~1 min on 16 cores).  Also: sum_I2
    equals the exact integer sum of squares, sampled residuals match, and the
    R-14 secondary metric 255 max|dK| is reported."""
    from oracle import parallel
    fr = video_c2.frames[:1800]
    fp = prnu.extract_fingerprint(fr, 1, batch=BENCH_BATCH)
    assert fp.n_sda == 1800
    sq = torch.zeros((1080, 1920), dtype=torch.int64, device="cuda")
    for i in range(0, 1800, 100):
        x = fr[i:i + 100].to(torch.int64)
        sq += (x * x).sum(0)
    assert torch.equal(fp.sum_I2, sq.double())                       # exact (all sums < 2^53)
    # residuals of sampled frames (same kernels, batch of 3)
    idx = [0, 977, 1799]
    Wg = prnu.residual(fr[idx].contiguous()).cpu().numpy()
    for j, i in enumerate(idx):
        Wr = oracle.residual(fr[i].cpu().numpy().astype(np.float32))
        assert np.abs(Wg[j] - Wr).max() <= W_TOL
    host = fr.cpu().numpy()
    K_ref, num, den, ns = parallel.extract_fingerprint_chunked(host, 1)
    assert ns == 1800
    np.testing.assert_array_equal(fp.sum_I2.cpu().numpy(), den)
    Kg = fp.K.cpu().numpy()
    prim = k_metric(Kg, K_ref, den, ns)
    sec = 255.0 * float(np.abs(Kg.astype(np.float64) - K_ref).max())
    rho = prnu.ncc(fp.K, video_c2.K).item()
    d_ncc = abs(rho - oracle.ncc(K_ref, video_c2.K.cpu().numpy()))
    parity_report(f"C2 d=1 full 1800 frames: R-14 primary {prim:.3e}, secondary 255*max|dK| {sec:.3e}, "
          f"|dNCC| {d_ncc:.2e}, NCC(K, K_true) {rho:.4f}")
    assert prim <= K_TOL
    assert d_ncc <= NCC_TOL
    assert rho > 0.9


def test_c2_query_pce(prnu, video_c2):
    """The bench's PCE leg: query frame 1800 against the depth-50 fingerprint."""
    fr = video_c2.frames
    fp = prnu.extract_fingerprint(fr[:1800], 50, batch=36)
    q = fr[1800:1801]
    R = prnu.residual(q, zero_mean=True)
    res = prnu.pce(R, prnu.pce_template(fp.K, q))
    K_ref, _, _, _ = oracle.extract_fingerprint(fr[:1800].cpu().numpy(), 50)
    qn = q[0].cpu().numpy()
    p_ref, peak_ref, _ = oracle.pce(oracle.residual(qn.astype(np.float32), zero_mean=True),
                                    oracle.pce_template(K_ref, qn))
    assert (res.peak_y.item(), res.peak_x.item()) == peak_ref == (0, 0)
    assert abs(res.pce.item() - p_ref) <= PCE_RTOL * abs(p_ref)
    assert res.decision().item()


def test_c5_depth_sweep_sampled(prnu):
    """Config 5 (3600 frames 1920x1080, shift recipe): every depth of the sweep
    runs; d = 3600 and d = 300 are checked against the oracle in full; the
    denoise counts follow floor(m/d)."""
    v = synth.video("shift", 3600, 1080, 1920, seed=0, device="cuda")
    fr = v.frames
    host = None
    for d in (1, 2, 5, 10, 25, 50, 100, 300, 3600):
        fp = prnu.extract_fingerprint(fr, d, batch=BENCH_BATCH if d == 1 else max(1, min(64, 3600 // d)))
        assert fp.n_sda == 3600 // d
        assert prnu.ncc(fp.K, v.K).item() > 0.5
        if d in (300, 3600):
            if host is None:
                host = fr.cpu().numpy()
            K_ref, num, den, ns = oracle.extract_fingerprint(host, d)
            np.testing.assert_array_equal(fp.sum_I2.cpu().numpy(), den)
            assert k_metric(fp.K.cpu().numpy(), K_ref, den, ns) <= K_TOL


def test_c3_stills_sampled(prnu):
    """Config 3 shape (4000x3000 luma stills): residual parity on one still, the
    depth-50 fingerprint of 200 stills against the oracle (4 SDA frames)."""
    Y, K_luma = synth.stills(200, 3000, 4000, seed=0, device="cuda")
    Wg = prnu.residual(Y[7:8].contiguous()).cpu().numpy()[0]
    Wr = oracle.residual(Y[7].cpu().numpy().astype(np.float32))
    assert np.abs(Wg - Wr).max() <= W_TOL
    fp = prnu.extract_fingerprint(Y, 50, batch=4)
    K_ref, num, den, ns = oracle.extract_fingerprint(Y.cpu().numpy(), 50)
    assert ns == 4
    assert k_metric(fp.K.cpu().numpy(), K_ref, den, ns) <= K_TOL
    for d in (1, 5, 10, 20):
        assert prnu.extract_fingerprint(Y, d, batch=BENCH_BATCH if d == 1 else 20).n_sda == 200 // d


def test_c4_camera_id_full(prnu):
    """Config 4: 64 cameras x 300 frames 1280x720, depth 30, 64 query residuals
    against 64 fingerprints (4096 PCEs).  Against the oracle (worker processes on
    every host core): all 64 fingerprints (R-14, sum_I2 bit-exact), all 64 query
    residuals, and a full column and row of the PCE matrix (query q vs camera 0,
    query 0 vs camera c: 127 pairs; R-19 tie rule).  Directional: diagonal > 60,
    off-diagonal FPR < 1%."""
    from oracle import parallel
    H, W, n = 720, 1280, 64
    Ks, queries = [], []
    with parallel.OraclePool() as pool:
        fps, dens = [], []
        for c in range(n):
            v = synth.video("drift", 301, H, W, seed=4, camera=c, device="cuda")
            fp = prnu.extract_fingerprint(v.frames[:300], 30, batch=10)
            Ks.append(fp.K.clone())
            dens.append(fp.sum_I2.cpu().numpy())
            queries.append(v.frames[300].clone())
            fps.append(pool.fingerprint(v.frames[:300].cpu().numpy(), 30))
        Iq = torch.stack(queries)
        R = prnu.residual(Iq, zero_mean=True)
        qn = Iq.cpu().numpy()
        rres = [pool.residual(qn[q]) for q in range(n)]
        K_ref = []
        for c in range(n):
            Kr, den, ns = fps[c].get()
            assert ns == 10
            np.testing.assert_array_equal(dens[c], den)
            assert k_metric(Ks[c].cpu().numpy(), Kr, den, ns) <= K_TOL, c
            K_ref.append(Kr)
        R_ref = [r.get() for r in rres]
        Rg = R.cpu().numpy()
        for q in range(n):
            assert np.abs(Rg[q] - R_ref[q]).max() <= W_TOL, q
        plan = prnu.PcePlan(H, W, n)
        plan.set_residual(R)
        M = np.zeros((n, n))
        PY = np.zeros((n, n), dtype=np.int64)
        PX = np.zeros((n, n), dtype=np.int64)
        for c in range(n):
            res = plan.match(prnu.pce_template(Ks[c], Iq))
            M[:, c] = res.pce.cpu().numpy()
            PY[:, c] = res.peak_y.cpu().numpy()
            PX[:, c] = res.peak_x.cpu().numpy()
        pairs = [(q, 0) for q in range(n)] + [(0, c) for c in range(1, n)]
        jobs = [pool.pce(R_ref[q], oracle.pce_template(K_ref[c], qn[q])) for q, c in pairs]
        worst = 0.0
        for (q, c), j in zip(pairs, jobs):
            p_ref, peak_ref, gap, C = j.get()
            gpk = (int(PY[q, c]), int(PX[q, c]))
            if gpk != peak_ref:
                assert gap < 1e-4, (q, c, gpk, peak_ref)
                p_ref = oracle.match.pce_from_surface(C, peak=gpk)[0]
            rel = abs(M[q, c] - p_ref) / (abs(p_ref) + 1e-3)
            worst = max(worst, rel)
            assert abs(M[q, c] - p_ref) <= PCE_RTOL * abs(p_ref) + 1e-3, (q, c, M[q, c], p_ref)
    print(f"\nC4: 64 fingerprints, 64 residuals and {len(pairs)} PCE pairs vs the oracle; "
          f"worst PCE relative difference {worst:.2e}")
    off = M[~np.eye(n, dtype=bool)]
    assert np.all(np.diag(M) > 60)
    assert np.mean(off > 60) < 0.01
