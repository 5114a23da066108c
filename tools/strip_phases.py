"""Phase breakdown of k_analysis_strip (needs a -DPRNU_STRIP_PROFILE build)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_04573_b200 as prnu
import synth
depth = int(os.environ.get("PHASE_DEPTH", "1"))   # 2: level 1 on the fp32 SDA-frame kernel
v = synth.video("drift", 128 * depth, 1080, 1920, seed=0, device="cuda")
ex = prnu.Extractor(1080, 1920, depth, batch=64)
ex(v.frames); torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 16)()
prnu._lib.prnu_debug_strip_profile(buf, 1)
ex(v.frames); torch.cuda.synchronize()
prnu._lib.prnu_debug_strip_profile(buf, 1)
names = ["thread loads (mirrored rows)", "row pass", "B1 wait", "column pass", "V0,V2 write", "B2 wait",
         "V1 write", "B3 wait", "H pass", "B4 wait", "carries, loop head", "TMA wait", "carries (manual blocks)",
         "edge fix-ups"]
tot = sum(buf[k] for k in range(14))
for k in range(14):
    print(f"{names[k]:32s} {100.0 * buf[k] / tot:6.2f}%  {buf[k] / 1e9:8.3f} Gcyc")
print(f"{'total':32s} {100.0:6.2f}%  {tot / 1e9:8.3f} Gcyc")
