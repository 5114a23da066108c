"""Pinned host -> device copy bandwidth (the e2e bound): one stream vs two streams."""
import torch, time
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for streams in (1, 2):
    ss = [torch.cuda.Stream() for _ in range(streams)]
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for r in range(4):
        chunk = n // streams
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"{streams} stream(s): {4 * n / dt / 1e9:.1f} GB/s")
