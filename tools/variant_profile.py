"""Per-pass times of the f3 variant residual (KTimer names of csrc/variant.cu), NB (argv[1], default 8) FHD frames."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_04573_b200 as prnu

NB = int(sys.argv[1]) if len(sys.argv) > 1 else 8
I = torch.rand((NB, 1080, 1920), device="cuda") * 255
for v in ((8, 0, 0), (16, 0, 0), (8, 1, 0), (8, 1, 1), (16, 1, 1)):
    var = prnu.DenoiseVariant(*v)
    out = torch.empty_like(I)
    prnu.residual_variant(I, var, out=out)
    torch.cuda.synchronize()
    prnu._lib.prnu_profile_begin()
    for _ in range(3):
        prnu.residual_variant(I, var, out=out)
    torch.cuda.synchronize()
    maxk = 32
    names = ctypes.create_string_buffer(64 * maxk)
    tot = (ctypes.c_double * maxk)()
    cnt = (ctypes.c_int64 * maxk)()
    nk = ctypes.c_int()
    prnu._lib.prnu_profile_end(maxk, names, tot, cnt, ctypes.byref(nk))
    rows = []
    for k in range(min(nk.value, maxk)):
        nm = names.raw[64 * k: 64 * k + 64].split(b"\0")[0].decode()
        rows.append((tot[k] / 3, cnt[k] / 3, nm))
    s = sum(r[0] for r in rows)
    print(f"== {v}: {s:.3f} ms per call of {NB} frames ({s / NB:.4f} ms/frame)")
    for t, c, nm in sorted(rows, reverse=True):
        print(f"   {nm:20s} {t:8.3f} ms  {c:5.1f} launches")
