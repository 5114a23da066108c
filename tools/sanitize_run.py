"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
every C-ABI entry point once, at small sizes (several tiles, ragged tails, odd
widths, unaligned frame pointers), plus one 2-frame FHD wave of the fused
extraction (u8, u16 SDA sums, fp32 SDA frames).  Kernel results are not checked
here (the GPU parity suite does that); the sanitizer reports hazards and errors.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py [--quick]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1909_04573_b200 as prnu  # noqa: E402
import synth  # noqa: E402

quick = "--quick" in sys.argv
dev = "cuda"
g = torch.Generator(device=dev)
g.manual_seed(7)


def u8(*shape):
    return torch.randint(0, 256, shape, dtype=torch.uint8, device=dev, generator=g)


steps = []


def step(name, fn):
    fn()
    torch.cuda.synchronize()
    steps.append(name)
    print("ok", name, flush=True)


# a1 SDA average (vector and scalar paths)
step("sda_average 8x64x128 d=4", lambda: prnu.sda_average(u8(8, 64, 128), 4))
step("sda_average 5x33x37 d=2", lambda: prnu.sda_average(u8(5, 33, 37), 2))
# a2-a4 residual: u8 / fp32, odd sizes, levels, window subsets, zero-mean
for (b, H, W) in ((2, 16, 16), (3, 37, 53), (2, 70, 131), (1, 130, 170)):
    step(f"residual u8 {b}x{H}x{W}", lambda b=b, H=H, W=W: prnu.residual(u8(b, H, W)))
    step(f"residual f32 {b}x{H}x{W} zm", lambda b=b, H=H, W=W: prnu.residual(u8(b, H, W).float(), zero_mean=True))
step("residual levels=1 windows(3,7)", lambda: prnu.residual(u8(2, 40, 48).float(),
                                                             prnu.DenoiseParams(levels=1, windows=(3, 7))))
step("residual levels=6", lambda: prnu.residual(u8(1, 96, 80).float(), prnu.DenoiseParams(levels=6)))
# a5-a6
W_ = prnu.residual(u8(3, 40, 56).float())
I_ = u8(3, 40, 56).float()
s1 = torch.zeros((40, 56), dtype=torch.float64, device=dev)
s2 = torch.zeros_like(s1)
step("fingerprint_accumulate", lambda: prnu.fingerprint_accumulate(W_, I_, s1, s2))
step("fingerprint_finalize", lambda: prnu.fingerprint_finalize(s1, s2 + 1.0))
# fused extraction: d = 1 (u8), 3 (u16 sums), 300 (fp32), odd width, unaligned frames, several waves
v = synth.video("shift", 24, 64, 64, seed=0, device=dev)
step("extract d=1", lambda: prnu.extract_fingerprint(v.frames, 1, batch=5))
step("extract d=3 (u16 sums)", lambda: prnu.extract_fingerprint(v.frames, 3, batch=3))
step("extract d=8 odd width", lambda: prnu.extract_fingerprint(u8(16, 45, 77), 8, batch=2))
step("extract d=1 unaligned frames", lambda: prnu.extract_fingerprint(u8(6 * 32 * 48 + 8)[8:].view(6, 32, 48), 1,
                                                                      batch=4))
step("extract d=300 (fp32 SDA)", lambda: prnu.extract_fingerprint(u8(600, 24, 40), 300, batch=2))
step("extract stride 3", lambda: prnu.extract_fingerprint_stride(v.frames, 3, batch=4))
step("GraphExtractor", lambda: prnu.GraphExtractor(24, 64, 64, 4, batch=3)(v.frames))
step("CameraBatchExtractor", lambda: prnu.CameraBatchExtractor(64, 64, 4, batch=3, streams=2)([v.frames] * 3))
hostfr = v.frames.cpu().pin_memory()
step("extract host", lambda: prnu.Extractor(64, 64, 4, batch=3, host=True)(hostfr))
step("multi host", lambda: prnu.MultiExtractor(24, 64, 64, (1, 4), batch=4)(hostfr))
# a7-a8
Ka = torch.randn(3, 48, 64, device=dev, generator=g)
step("ncc", lambda: prnu.ncc(Ka, Ka * 2 + 1))
Rq = prnu.residual(u8(2, 48, 64), zero_mean=True)
Tq = prnu.pce_template(Ka[0], u8(2, 48, 64))
step("pce", lambda: prnu.pce(Rq, Tq))
step("pce aligned", lambda: prnu.pce(Rq, Tq, aligned=True))
plan = prnu.PcePlan(48, 64, 2)
plan.set_residual(Rq)
step("pce cached", lambda: plan.match(Tq))
# NEXT rows
step("block_match 130x170/50", lambda: prnu.block_match(torch.randn(130, 170, device=dev, generator=g),
                                                         torch.randn(130, 170, device=dev, generator=g), 50))
K0 = prnu.extract_fingerprint(v.frames, 4, batch=4).K
step("wdft", lambda: prnu.wdft(torch.stack([K0, K0])))
step("rgb_to_luma planar", lambda: prnu.rgb_to_luma(u8(2, 3, 16, 24)))
step("rgb_to_luma interleaved u8", lambda: prnu.rgb_to_luma(u8(2, 16, 24, 3), "interleaved", torch.uint8))
for taps, bnd, tr in ((16, 0, 0), (8, 1, 0), (16, 1, 0), (8, 1, 1), (16, 1, 1)):
    step(f"variant taps={taps} boundary={bnd} transform={tr}",
         lambda taps=taps, bnd=bnd, tr=tr: prnu.residual_variant(u8(2, 40, 52).float(),
                                                                 prnu.DenoiseVariant(taps, bnd, tr)))
# one FHD wave of the fused extraction: u8 frames, u16 SDA sums
if not quick:
    fhd = synth.video("drift", 4, 1080, 1920, seed=0, device=dev).frames
    step("FHD extract d=1 (2-frame waves)", lambda: prnu.extract_fingerprint(fhd, 1, batch=2))
    step("FHD extract d=2 (u16 sums)", lambda: prnu.extract_fingerprint(fhd, 2, batch=2))
    step("FHD residual f32 1 frame", lambda: prnu.residual(fhd[:1].float()))
print(f"sanitize workload: {len(steps)} steps done", flush=True)
