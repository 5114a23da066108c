"""u8 residual (TMA analysis path) vs the same frames as fp32 (generic path): must be bit-identical."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1909_04573_b200 as prnu  # noqa: E402

H = int(sys.argv[1]) if len(sys.argv) > 1 else 1080
W = int(sys.argv[2]) if len(sys.argv) > 2 else 1920
b = int(sys.argv[3]) if len(sys.argv) > 3 else 1
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randint(0, 256, (b, H, W), generator=g, device="cuda", dtype=torch.uint8)
w8 = prnu.residual(x)
torch.cuda.synchronize()
wf = prnu.residual(x.float())
torch.cuda.synchronize()
print("max diff u8 vs f32", (w8 - wf).abs().max().item(), "equal", torch.equal(w8, wf))
