"""Small driver for ncu: depth-1 extraction of a few Full-HD frames (+ one depth-50 group)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1909_04573_b200 as prnu  # noqa: E402
import synth  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 64
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 16
v = synth.video("drift", m, 1080, 1920, seed=0, device="cuda")
ex = prnu.Extractor(1080, 1920, 1, batch=batch)
for _ in range(2):
    fp = ex(v.frames)
ex50 = prnu.Extractor(1080, 1920, 50, batch=max(1, m // 50))
if m >= 50:
    ex50(v.frames)
torch.cuda.synchronize()
print("ok", fp.n_sda, prnu.ncc(fp.K, v.K).item())
