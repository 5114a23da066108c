"""prnu.residual throughput (fp32 and u8 FHD planes, batch 64)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_04573_b200 as prnu
for dt in (torch.uint8, torch.float32):
    x = (torch.rand((64, 1080, 1920), device="cuda") * 255).to(dt)
    out = torch.empty((64, 1080, 1920), device="cuda")
    prnu.residual(x, out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        prnu.residual(x, out=out)
    b.record()
    torch.cuda.synchronize()
    print(dt, "%.3f ms per 64 frames" % (a.elapsed_time(b) / 5))
