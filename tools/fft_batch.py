"""cuFFT R2C + C2R time per 720x1280 transform pair vs batch size (camera-ID PCE cost)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_04573_b200 as prnu

H, W = 720, 1280
for b in (16, 64, 128, 256):
    R = torch.randn(b, H, W, device="cuda")
    T = torch.randn(b, H, W, device="cuda")
    plan = prnu.PcePlan(H, W, b)
    plan.set_residual(R)
    plan.match(T)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(2, 512 // b)
    e0.record()
    for _ in range(reps):
        plan.match(T)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"batch {b:4d}: {ms:8.3f} ms per call, {1000 * ms / b:7.2f} us per pair")
    del plan, R, T
    torch.cuda.empty_cache()
