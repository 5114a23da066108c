"""f3 denoiser variants: GPU (prnu_residual_variant through the C ABI) vs the fp64
oracle (oracle/variants.py) on the same seeded inputs.  Tolerance as the default
residual: max |dW| <= 1e-3 intensity units (BASELINE north_star)."""
import numpy as np
import pytest
import torch

from oracle import variants as V

pytestmark = pytest.mark.gpu

W_TOL = 1e-3
# (GPU variant fields, oracle keyword arguments)
VARIANTS = [((8, 0, 0), dict()), ((16, 0, 0), dict(taps=16)), ((8, 1, 0), dict(boundary=1)),
            ((16, 1, 0), dict(taps=16, boundary=1)), ((8, 1, 1), dict(transform=1)),
            ((16, 1, 1), dict(taps=16, transform=1))]
IDS = ["db4-sym", "db8-sym", "db4-per", "db8-per", "db4-swt", "db8-swt"]


@pytest.fixture(scope="module")
def prnu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1909_04573_b200 as m
    return m


def _textured(b, H, W, seed):
    g = np.random.default_rng(seed)
    y, x = np.mgrid[0:H, 0:W]
    out = []
    for _ in range(b):
        f = 128 + 50 * np.sin(2 * np.pi * (x / g.uniform(5, 40) + y / g.uniform(5, 40)))
        f += 20 * np.cos(2 * np.pi * y / g.uniform(3, 9)) + g.normal(0, 4, (H, W))
        out.append(np.clip(f, 0, 255))
    return np.stack(out).astype(np.float32)


@pytest.mark.parametrize("v,kw", VARIANTS, ids=IDS)
@pytest.mark.parametrize("b,H,W", [(1, 64, 64), (2, 37, 53), (1, 135, 240), (1, 16, 16), (1, 100, 333)])
def test_variant_matches_oracle(prnu, v, kw, b, H, W):
    I = _textured(b, H, W, H * W + b + v[0])
    got = prnu.residual_variant(torch.from_numpy(I).cuda(), prnu.DenoiseVariant(*v)).cpu().numpy()
    for i in range(b):
        err = np.abs(got[i] - V.residual(I[i], **kw)).max()
        assert err <= W_TOL, (i, err)


@pytest.mark.parametrize("v,kw", VARIANTS[1:], ids=IDS[1:])
@pytest.mark.parametrize("levels,windows,s0", [(1, (3,), 9.0), (3, (5, 9), 4.0), (6, (3, 5, 7, 9), 25.0)])
def test_variant_params_match_oracle(prnu, v, kw, levels, windows, s0):
    I = _textured(1, 96, 130, levels)[0]
    p = prnu.DenoiseParams(sigma0_sq=s0, levels=levels, windows=windows)
    got = prnu.residual_variant(torch.from_numpy(I).cuda(), prnu.DenoiseVariant(*v), p).cpu().numpy()
    ref = V.residual(I, sigma0_sq=s0, windows=windows, levels=levels, **kw)
    assert np.abs(got - ref).max() <= W_TOL


def test_default_variant_equals_fast_path(prnu):
    """{8, symmetric, decimated} through the generic passes == the fused default path, up to
    fp32 rounding order (both are within W_TOL of the oracle; measured 3e-4)."""
    I = torch.from_numpy(_textured(3, 135, 240, 9)).cuda()
    a = prnu.residual_variant(I, prnu.DenoiseVariant())
    b = prnu.residual(I)
    assert (a - b).abs().max().item() <= W_TOL


@pytest.mark.parametrize("v,kw", VARIANTS[1:], ids=IDS[1:])
def test_variant_zero_mean_and_invariants(prnu, v, kw):
    I = np.round(_textured(2, 70, 90, 11))
    Ig = torch.from_numpy(I).cuda()
    var = prnu.DenoiseVariant(*v)
    got = prnu.residual_variant(Ig, var, zero_mean=True).cpu().numpy()
    for i in range(2):
        assert np.abs(got[i] - V.residual(I[i], zero_mean=True, **kw)).max() <= W_TOL
        assert np.abs(got[i].astype(np.float64).mean(axis=0)).max() < 1e-4
    c = torch.full((1, 64, 96), 128.0, device="cuda")
    assert prnu.residual_variant(c, var).abs().max().item() < 1e-4
    d = prnu.residual_variant(Ig + 10.0, var) - prnu.residual_variant(Ig, var)
    assert d.abs().max().item() < 1e-3


def test_variant_deterministic_and_batch_independent(prnu):
    I = torch.from_numpy(_textured(4, 64, 80, 3)).cuda()
    for v in ((16, 1, 0), (8, 1, 1)):
        var = prnu.DenoiseVariant(*v)
        a = prnu.residual_variant(I, var)
        b = prnu.residual_variant(I, var)
        c = torch.cat([prnu.residual_variant(I[i:i + 1], var) for i in range(4)])
        assert torch.equal(a, b) and torch.equal(a, c)


def test_variant_errors(prnu):
    I = torch.zeros((1, 64, 64), device="cuda")
    with pytest.raises(prnu.PrnuError) as e:
        prnu.residual_variant(I, prnu.DenoiseVariant(8, 0, 1))      # undecimated must be circular
    assert e.value.code == 4
    with pytest.raises(prnu.PrnuError) as e:
        prnu.residual_variant(I, prnu.DenoiseVariant(10, 0, 0))
    assert e.value.code == 4
    with pytest.raises(prnu.PrnuError) as e:
        prnu.residual_variant(torch.zeros((1, 15, 64), device="cuda"), prnu.DenoiseVariant(16, 1, 0))
    assert e.value.code == 2


@pytest.mark.parametrize("v,kw", VARIANTS[1:], ids=IDS[1:])
def test_variant_full_hd(prnu, v, kw):
    """BASELINE configs[1] frame size (1080 x 1920), one frame, every output."""
    I = _textured(1, 1080, 1920, 77)
    got = prnu.residual_variant(torch.from_numpy(I).cuda(), prnu.DenoiseVariant(*v)).cpu().numpy()[0]
    assert np.abs(got - V.residual(I[0], **kw)).max() <= W_TOL


@pytest.mark.parametrize("v,kw", [VARIANTS[0], VARIANTS[3], VARIANTS[5]], ids=[IDS[0], IDS[3], IDS[5]])
@pytest.mark.parametrize("depth", [1, 4])
def test_variant_fingerprint_matches_oracle(prnu, v, kw, depth):
    """f3 fingerprint (SDA -> variant residual -> MLE -> finalize) vs the oracle's
    composition of the same steps; R-14 metric <= 1e-3 (as the default path)."""
    import oracle
    g = torch.Generator().manual_seed(5 + depth)
    fr = torch.randint(20, 236, (16, 64, 80), generator=g, dtype=torch.uint8)
    fp = prnu.extract_fingerprint_variant(fr.cuda(), depth, prnu.DenoiseVariant(*v), batch=3)
    S = oracle.sda_average(fr.numpy(), depth)
    num = np.zeros((64, 80))
    den = np.zeros((64, 80))
    for i in range(S.shape[0]):
        oracle.mle_accumulate(V.residual(S[i], **kw), S[i], num, den)
    K = oracle.finalize(num, den)
    assert fp.n_sda == S.shape[0]
    np.testing.assert_array_equal(fp.sum_I2.cpu().numpy(), den)     # exact fp64 sums of exact products
    d = np.abs(fp.K.cpu().numpy().astype(np.float64) - K)
    assert float((d * np.sqrt(den / S.shape[0])).max()) <= W_TOL


@pytest.mark.parametrize("v", [(16, 0, 0), (8, 1, 0), (8, 1, 1)])
@pytest.mark.parametrize("m,depth,batch", [(16, 4, 3), (23, 2, 5)])
def test_variant_extraction_is_the_composition(prnu, v, m, depth, batch):
    """prnu_extract_fingerprint_variant (native waves) is bit-identical to composing
    prnu_sda_average -> prnu_residual_variant -> prnu_fingerprint_accumulate ->
    prnu_fingerprint_finalize over the same waves (remainder frames dropped)."""
    g = torch.Generator().manual_seed(m + depth)
    fr = torch.randint(0, 256, (m, 48, 72), generator=g, dtype=torch.uint8).cuda()
    var = prnu.DenoiseVariant(*v)
    fp = prnu.extract_fingerprint_variant(fr, depth, var, batch=batch)
    ns = m // depth
    s_wi = torch.zeros((48, 72), dtype=torch.float64, device="cuda")
    s_i2 = torch.zeros_like(s_wi)
    for g0 in range(0, ns, batch):
        g1 = min(g0 + batch, ns)
        S = prnu.sda_average(fr[g0 * depth: g1 * depth], depth)
        Wr = prnu.residual_variant(S, var)
        prnu.fingerprint_accumulate(Wr, S, s_wi, s_i2)
    K = prnu.fingerprint_finalize(s_wi, s_i2, 1e-6)
    assert fp.n_sda == ns
    assert torch.equal(fp.sum_WI, s_wi) and torch.equal(fp.sum_I2, s_i2) and torch.equal(fp.K, K)
