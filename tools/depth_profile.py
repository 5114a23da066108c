"""Kernel breakdown of one fingerprint extraction at a given depth (FHD, 1800 frames)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_04573_b200 as prnu
import synth

d = int(sys.argv[1]) if len(sys.argv) > 1 else 2
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 64
m, H, W = 1800, 1080, 1920
v = synth.video("drift", m, H, W, seed=0, device="cuda")
ex = prnu.Extractor(H, W, d, batch)
ex(v.frames)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); ex(v.frames); b.record(); torch.cuda.synchronize()
print(f"depth {d} batch {batch}: {a.elapsed_time(b):.2f} ms for {m // d} SDA frames")
prnu._lib.prnu_profile_begin()
ex(v.frames)
torch.cuda.synchronize()
maxk = 32
names = ctypes.create_string_buffer(64 * maxk)
tot = (ctypes.c_double * maxk)()
cnt = (ctypes.c_int64 * maxk)()
nk = ctypes.c_int()
prnu._lib.prnu_profile_end(maxk, names, tot, cnt, ctypes.byref(nk))
rows = sorted(((tot[k], cnt[k], names.raw[64 * k: 64 * k + 64].split(b"\0")[0].decode()) for k in range(nk.value)),
              reverse=True)
for t, c, nm in rows:
    print(f"   {nm:20s} {t:8.3f} ms  {c:4d} launches  {t * 1000 / (m // d):7.2f} us/SDA frame")
