"""Extraction speed for u8 widths with / without 16-byte-aligned rows (TMA vs thread-loaded staging)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_04573_b200 as prnu
for H, W in ((1080, 1920), (1080, 1919), (768, 1366), (768, 1376)):
    fr = torch.randint(0, 256, (360, H, W), dtype=torch.uint8, device="cuda")
    ex = prnu.Extractor(H, W, 1, 360)
    ex(fr)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        ex(fr)
    b.record()
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / 3
    print(f"{H}x{W}: {t:.2f} ms for 360 frames, {t * 1000 / 360 / (H * W / 2.0736e6):.2f} us per FHD-equivalent frame")
