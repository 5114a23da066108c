import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, ctypes
import paper_1909_04573_b200 as prnu
from scipy.ndimage import uniform_filter
H, W = 16, 24
rng = np.random.default_rng(H * W)
y, x = np.mgrid[0:H, 0:W]
K = rng.normal(0, 0.01, (H, W)) + 0.03 * np.cos(2 * np.pi * (3 * y / H + 7 * x / W))
K = (K - K.mean()).astype(np.float32)
plan = prnu.WdftPlan(H, W, 1)
out = plan(torch.from_numpy(K).cuda()).cpu().numpy()
torch.cuda.synchronize()
ws = plan.ws.view(torch.uint8)
# layout: work, F, A, Ahat, part, s2  (mirror run_wdft)
def al(n): return (n + 255) // 256 * 256
import struct
# we don't know cuFFT work size: recompute offsets from the end: s2 is last
P = H * W; nf = W // 2 + 1
tot = plan.nbytes
s2_off = tot - al(4 * 1)
part_off = s2_off - al(8 * 148)
ahat_off = part_off - al(4 * P)
a_off = ahat_off - al(4 * P)
A = ws[a_off:a_off + 4 * P].cpu().numpy().view(np.float32).reshape(H, W)
Ah = ws[ahat_off:ahat_off + 4 * P].cpu().numpy().view(np.float32).reshape(H, W)
s2 = ws[s2_off:s2_off + 4].cpu().numpy().view(np.float32)[0]
Kd = K.astype(np.float64)
F = np.fft.fft2(Kd)
A_ref = np.abs(F) / np.sqrt(P)
s2_ref = np.mean(Kd * Kd)
m = np.full((H, W), np.inf)
for w in (3, 5, 7, 9):
    m = np.minimum(m, uniform_filter(A_ref ** 2, size=w, mode="reflect"))
Ah_ref = A_ref * s2_ref / np.maximum(m, s2_ref)
print("s2", s2, s2_ref)
print("A err", np.max(np.abs(A - A_ref)) / A_ref.max())
print("Ahat err", np.max(np.abs(Ah - Ah_ref)) / Ah_ref.max())
i = np.unravel_index(np.argmax(np.abs(Ah - Ah_ref)), Ah.shape); print("worst at", i, Ah[i], Ah_ref[i], A[i], A_ref[i])
