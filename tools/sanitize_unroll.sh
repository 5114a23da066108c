cd /root/repo
PRNU_NVCC_DEFS="PRNU_H_UNROLL=3" python paper_1909_04573_b200/_build.py --force > /dev/null 2>&1
cat > /tmp/t.py <<'PY'
import sys; sys.path.insert(0, "/root/repo")
import torch, paper_1909_04573_b200 as prnu
for (h, w) in [(64, 64), (300, 520), (1080, 1920)]:
    x = (torch.rand(2, h, w, device="cuda") * 255)
    r = prnu.residual(x); torch.cuda.synchronize(); print("ok f32", h, w, float(r.abs().max()), flush=True)
x = (torch.rand(200, 1080, 1920, device="cuda") * 255).to(torch.uint8)
ex = prnu.Extractor(1080, 1920, 50, batch=4); fp = ex(x); torch.cuda.synchronize(); print("ok d50", flush=True)
ex = prnu.Extractor(1080, 1920, 1, batch=64); fp = ex(x); torch.cuda.synchronize(); print("ok d1", flush=True)
PY
timeout 300 python /tmp/t.py 2>&1 | tail -5
python paper_1909_04573_b200/_build.py --force > /dev/null 2>&1
