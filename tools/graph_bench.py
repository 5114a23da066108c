import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, torch, paper_1909_04573_b200 as prnu
def timeit(fn, n=20):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e3
for (m, H, W, d, b) in [(16, 64, 64, 4, 16), (16, 64, 64, 1, 16), (300, 720, 1280, 30, 16), (64, 270, 480, 1, 64)]:
    g = torch.Generator(device="cpu").manual_seed(1)
    fr = torch.randint(0, 256, (m, H, W), generator=g, dtype=torch.uint8).cuda()
    ex = prnu.Extractor(H, W, d, b)
    gx = prnu.GraphExtractor(m, H, W, d, b)
    a = ex(fr).K.clone(); c = gx(fr).K.clone()
    print((m, H, W, d), "equal", torch.equal(a, c), "eager %.3f ms graph %.3f ms" % (timeit(lambda: ex(fr)), timeit(lambda: gx())))
