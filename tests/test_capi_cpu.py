"""The C-ABI library loads and exports every symbol include/prnu.h declares;
host-side validation and workspace queries work without a GPU (no compute)."""
import ctypes
import os

import numpy as np

import pytest

import paper_1909_04573_b200 as prnu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    syms = prnu.header_symbols()
    assert len(syms) >= 20
    lib = ctypes.CDLL(prnu.LIB_PATH)
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", prnu.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_default_params_and_version():
    p = prnu._Params()
    assert prnu._lib.prnu_default_params(ctypes.byref(p)) == 0
    assert abs(p.sigma0_sq - 9.0) < 1e-7 and p.levels == 4 and p.n_windows == 4
    assert list(p.windows) == [3, 5, 7, 9]
    assert "sm_100a" in prnu.version()


def test_sda_groups_host():
    # P:436 counts via the library's host-side planner
    assert [prnu.sda_groups(1200, d) for d in (1, 5, 10, 30, 50, 200, 1200)] == [1200, 240, 120, 40, 24, 6, 1]
    with pytest.raises(prnu.PrnuError) as e:
        prnu.sda_groups(10, 11)
    assert e.value.code == 3


def test_validation_is_synchronous_and_precedes_launch():
    p = prnu.DenoiseParams().c()
    L = prnu._lib
    # null pointers -> INVALID_ARG
    assert L.prnu_residual(None, 1, 64, 64, ctypes.byref(p), 0, None, None, 0, None) == 1
    # plane too small
    dummy = ctypes.c_void_p(1 << 20)
    assert L.prnu_residual(dummy, 1, 15, 64, ctypes.byref(p), 0, dummy, dummy, 1 << 30, None) == 2
    # bad parameter
    bad = prnu.DenoiseParams(windows=(4,)).c()
    assert L.prnu_residual(dummy, 1, 64, 64, ctypes.byref(bad), 0, dummy, dummy, 1 << 30, None) == 4
    bad = prnu.DenoiseParams(sigma0_sq=0.0).c()
    assert L.prnu_residual(dummy, 1, 64, 64, ctypes.byref(bad), 0, dummy, dummy, 1 << 30, None) == 4
    # workspace too small
    assert L.prnu_residual(dummy, 1, 64, 64, ctypes.byref(p), 0, dummy, dummy, 16, None) == 9
    # prnu_check_results: argument validation before any device work
    assert L.prnu_check_results(3, dummy, 10, None) == 1
    assert L.prnu_check_results(0, dummy, 0, None) == 1
    assert L.prnu_check_results(0, None, 10, None) == 1
    # workspace not 256-byte aligned (the header's contract; the pyramid is written with 256-bit stores)
    off = ctypes.c_void_p((1 << 20) + 16)
    assert L.prnu_residual(dummy, 1, 64, 64, ctypes.byref(p), 0, dummy, off, 1 << 30, None) == 1
    K = ctypes.c_void_p(1 << 21)
    assert L.prnu_extract_fingerprint(dummy, 16, 64, 64, 4, ctypes.byref(p), 4, ctypes.c_double(1e-6), K, K, K, None,
                                      off, ctypes.c_size_t(1 << 30), None) == 1
    # depth exceeds frames
    assert L.prnu_sda_average(dummy, 10, 8, 8, 11, dummy, None, None) == 3
    assert "depth" in L.prnu_last_error().decode()


def test_workspace_queries():
    p = prnu.DenoiseParams().c()
    L = prnu._lib
    a = L.prnu_residual_workspace_bytes(1, 1080, 1920, ctypes.byref(p))
    b = L.prnu_residual_workspace_bytes(8, 1080, 1920, ctypes.byref(p))
    assert a > 1080 * 1920 * 4 and b > 7 * (a - L.prnu_finalize_workspace_bytes(1080, 1920))
    assert L.prnu_extract_workspace_bytes(1080, 1920, 16, 50, ctypes.byref(p)) > \
        L.prnu_extract_workspace_bytes(1080, 1920, 16, 1, ctypes.byref(p))
    assert L.prnu_residual_workspace_bytes(1, 8, 8, ctypes.byref(p)) == 0   # 8 < 2^4


def test_variant_filters_match_oracle_factorisation():
    """f3: the library's 8- and 16-tap lowpass (fp32 constants, host call) equal the
    oracle's spectral factorisation (minimum-phase order = reversed dec_lo) to fp32 rounding."""
    import numpy as np
    from oracle import variants as V
    for taps, p in ((8, 4), (16, 8)):
        got = np.array(prnu.wavelet_filter(taps))
        ref = V.daubechies(p)[::-1]
        assert np.abs(got - ref.astype(np.float32).astype(np.float64)).max() == 0.0, taps
    with pytest.raises(prnu.PrnuError) as e:
        prnu.wavelet_filter(12)
    assert e.value.code == 4


def test_variant_validation_host():
    """Variant fields are validated before any launch (workspace query returns 0)."""
    p = prnu.DenoiseParams().c()
    for v, ok in (((8, 0, 0), True), ((16, 1, 0), True), ((8, 1, 1), True), ((16, 1, 1), True),
                  ((12, 0, 0), False), ((8, 2, 0), False), ((8, 0, 1), False), ((8, 0, 2), False)):
        vv = prnu.DenoiseVariant(*v).c()
        n = prnu._lib.prnu_residual_variant_workspace_bytes(2, 64, 96, ctypes.byref(p), ctypes.byref(vv))
        assert (n > 0) == ok, v


def test_lifting_constants_reproduce_the_filter():
    """R-27: the lifting constants compiled into analysis.cu (LF_*) are those of the
    factorisation in tools/lifting.py (to fp32 precision) and, used in fp64, the
    cascade reproduces R-2's direct analysis filter pair to rounding."""
    import importlib.util
    import re
    src = open(os.path.join(ROOT, "paper_1909_04573_b200", "csrc", "analysis.cu")).read()
    lf = {m.group(1): float(m.group(2)) for m in re.finditer(r"#define (LF_\w+) ([-0-9.e]+)f", src)}
    spec = importlib.util.spec_from_file_location("lifting", os.path.join(ROOT, "tools", "lifting.py"))
    L = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(L)
    M, steps = L.factor()
    q1, q2, q3, q4 = [s_[2] for s_ in steps]
    KA, KD = M[0][1][1][0], M[1][0][1][0]
    want = {"LF_C1": q1[1][0], "LF_C2A": -q2[1][0], "LF_C2B": q2[1][1], "LF_C3A": -q3[1][0], "LF_C3B": q3[1][1],
            "LF_C4A": -q4[1][0], "LF_C4B": -q4[1][1], "LF_C5": -M[1][1][1][0] / KD, "LF_KA": KA, "LF_KD": KD,
            "LF_KA2": KA * KA, "LF_KD2": KD * KD, "LF_KD4": KD ** 4}
    for k, v in want.items():
        assert np.float32(lf[k]) == np.float32(v), (k, lf[k], v)
    x = np.random.default_rng(3).uniform(0, 255, 256)
    c = [lf[k] for k in ("LF_C1", "LF_C2A", "LF_C2B", "LF_C3A", "LF_C3B", "LF_C4A", "LF_C4B", "LF_C5", "LF_KA",
                         "LF_KD")]
    assert np.abs(L.lift(x, *c, np.float64) - L.direct(x, np.float64)).max() < 1e-11


def test_sda_division_sequence_exact():
    """R-28: q = RN(q0 + RN(s - q0 d) r), q0 = RN(s r), r = RN(1/d) equals the correctly
    rounded fp32 quotient s/d for every integer s <= 255 d (a subset of depths here;
    tools/sda_div_check.py runs every d <= 257 and the config depths)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("sda_div_check", os.path.join(ROOT, "tools", "sda_div_check.py"))
    D = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(D)
    for d in (2, 3, 5, 7, 10, 25, 30, 50, 100, 255, 256, 257):
        assert D.check(d) == 0, d


def test_extract_variant_workspace_validation():
    """prnu_extract_variant_workspace_bytes: > 0 for valid arguments, 0 for a bad
    variant, batch or plane (validated on the host before any launch)."""
    p = prnu.DenoiseParams().c()
    L = prnu._lib
    ok = prnu.DenoiseVariant(16, 0, 0).c()
    bad = prnu.DenoiseVariant(12, 0, 0).c()
    assert L.prnu_extract_variant_workspace_bytes(64, 96, 4, ctypes.byref(p), ctypes.byref(ok)) > 0
    assert L.prnu_extract_variant_workspace_bytes(64, 96, 4, ctypes.byref(p), ctypes.byref(bad)) == 0
    assert L.prnu_extract_variant_workspace_bytes(64, 96, 0, ctypes.byref(p), ctypes.byref(ok)) == 0
    assert L.prnu_extract_variant_workspace_bytes(0, 96, 4, ctypes.byref(p), ctypes.byref(ok)) == 0
