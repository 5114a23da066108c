"""One cached PCE call of 64 720x1280 pairs per variant (for an ncu launch list):
match(T) and match_template(K, Iq)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_04573_b200 as prnu
H, W, b = 720, 1280, 64
R = torch.randn(b, H, W, device="cuda")
T = torch.randn(b, H, W, device="cuda")
K = torch.randn(H, W, device="cuda")
Iq = torch.randint(0, 256, (b, H, W), dtype=torch.uint8, device="cuda")
plan = prnu.PcePlan(H, W, b)
plan.set_residual(R)
for _ in range(2):
    plan.match(T)
    plan.match_template(K, Iq)
torch.cuda.synchronize()
print("ok")
