"""The C ABI used from plain C (examples/c_abi_extract.c: cudaMalloc + include/prnu.h,
no Python or torch on that path) gives the bits the Python binding gives."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1909_04573_b200")
CUDA = "/usr/local/cuda"


def build_example(out_dir):
    exe = os.path.join(out_dir, "c_abi_extract")
    cmd = ["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-I", CUDA + "/include",
           os.path.join(ROOT, "examples", "c_abi_extract.c"), "-L", LIBDIR, "-lprnu", "-L", CUDA + "/lib64",
           "-lcudart", "-Wl,-rpath," + LIBDIR, "-Wl,-rpath," + CUDA + "/lib64", "-o", exe]
    subprocess.check_call(cmd)
    return exe


def test_c_example_builds(tmp_path):
    """Compile-only (no GPU needed): the header is valid C and the library links."""
    assert os.path.exists(build_example(str(tmp_path)))


@pytest.mark.gpu
@pytest.mark.parametrize("m,H,W,d", [(16, 64, 64, 4), (30, 135, 240, 1)])
def test_c_example_matches_python_binding(tmp_path, m, H, W, d):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1909_04573_b200 as prnu
    exe = build_example(str(tmp_path))
    fr = np.random.default_rng(m + d).integers(0, 256, (m, H, W), dtype=np.uint8)
    fpath, kpath, rpath = (str(tmp_path / n) for n in ("frames.u8", "K.f32", "ref.f32"))
    fr.tofile(fpath)
    ref = prnu.extract_fingerprint(torch.from_numpy(fr).cuda(), d, batch=16).K.cpu().numpy()
    other = np.random.default_rng(7).standard_normal((H, W)).astype(np.float32)
    other.tofile(rpath)
    out = subprocess.run([exe, fpath, str(m), str(H), str(W), str(d), kpath, rpath], capture_output=True, text=True,
                         timeout=120)
    assert out.returncode == 0, out.stderr
    K = np.fromfile(kpath, dtype=np.float32).reshape(H, W)
    np.testing.assert_array_equal(K.view(np.uint32), ref.view(np.uint32))
    rho = float(out.stdout.split("ncc")[1].split()[0])
    rho_py = float(prnu.ncc(torch.from_numpy(ref).cuda(), torch.from_numpy(other).cuda()))
    assert rho == rho_py   # same kernel, same inputs
    assert int(out.stdout.split("launches")[1].split()[0]) > 0
