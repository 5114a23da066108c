import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_04573_b200 as prnu
H = int(sys.argv[1]) if len(sys.argv) > 1 else 64
W = int(sys.argv[2]) if len(sys.argv) > 2 else 64
x = torch.rand((1, H, W), device="cuda") * 255
w = prnu.residual(x)
torch.cuda.synchronize()
print("ok", w.abs().max().item())
