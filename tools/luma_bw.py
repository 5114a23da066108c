import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_1909_04573_b200 as prnu
H, W = 1080, 1920
for n in (16, 64):
    rgb = torch.randint(0, 256, (n, 3, H, W), dtype=torch.uint8, device="cuda")
    out = torch.empty((n, H, W), dtype=torch.float32, device="cuda")
    for dt in (torch.float32, torch.uint8):
        prnu.rgb_to_luma(rgb, dtype=dt); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10): prnu.rgb_to_luma(rgb, dtype=dt)
        b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        by = n * H * W * (3 + (4 if dt == torch.float32 else 1))
        print(n, dt, f"{ms:.3f} ms {by / ms / 1e6:.0f} GB/s")
