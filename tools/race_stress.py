"""Race evidence without compute-sanitizer (closed on the GPU pool): the outputs of a
fixed workload from the release build are saved, then recomputed by a build with
-DPRNU_RACE_STRESS (random warp delays at every barrier / mbarrier phase of the
shared-memory kernels, common.cuh) and -DPRNU_DEBUG (device bounds checks that trap),
and must be bit-identical.

    python tools/race_stress.py save|compare gpurun_out/race_ref.pt"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1909_04573_b200 as prnu  # noqa: E402
import synth  # noqa: E402
import time  # noqa: E402

mode, path = sys.argv[1], sys.argv[2]
print("library:", prnu.version())
dev = "cuda"
g = torch.Generator(device=dev)
g.manual_seed(11)


def u8(*shape):
    return torch.randint(0, 256, shape, dtype=torch.uint8, device=dev, generator=g)


t0 = time.perf_counter()
out = {}
for (b, H, W) in ((2, 16, 16), (3, 37, 53), (2, 70, 131), (2, 130, 170), (1, 1080, 1920)):
    x = u8(b, H, W)
    out[f"res_u8_{b}x{H}x{W}"] = prnu.residual(x)
    out[f"res_f32_{b}x{H}x{W}"] = prnu.residual(x.float() * 0.5, zero_mean=True)
out["res_l6"] = prnu.residual(u8(1, 96, 80).float(), prnu.DenoiseParams(levels=6))
out["res_w37"] = prnu.residual(u8(2, 40, 48).float(), prnu.DenoiseParams(levels=2, windows=(3, 7)))
v = synth.video("drift", 40, 270, 480, seed=1, device=dev)
for d, bt in ((1, 7), (3, 4), (20, 2)):
    fp = prnu.extract_fingerprint(v.frames, d, batch=bt)
    out[f"fp_d{d}_K"], out[f"fp_d{d}_num"], out[f"fp_d{d}_den"] = fp.K, fp.sum_WI, fp.sum_I2
fp = prnu.extract_fingerprint(u8(600, 24, 40), 300, batch=2)
out["fp_d300_K"] = fp.K
fp = prnu.extract_fingerprint(u8(9, 45, 77), 1, batch=4)
out["fp_odd_K"] = fp.K
fhd = synth.video("drift", 4, 1080, 1920, seed=0, device=dev).frames
out["fp_fhd_d1"] = prnu.extract_fingerprint(fhd, 1, batch=2).sum_WI
out["fp_fhd_d2"] = prnu.extract_fingerprint(fhd, 2, batch=2).sum_WI
R = prnu.residual(v.frames[:2], zero_mean=True)
T = prnu.pce_template(out["fp_d3_K"], v.frames[:2])
r = prnu.pce(R, T)
out["pce"], out["pce_y"], out["pce_x"] = r.pce, r.peak_y, r.peak_x
pb, nb = prnu.block_match(R[0], T[0], 100)
out["blk_pce"], out["blk_ncc"] = pb, nb
# the PCE row / column FFT kernels (pcefft.cu): 720p cached + fused templates, H = 96 with
# a row plan, H = 45 with cuFFT rows, 500 x 500 block tiles
Iq = u8(3, 720, 1280)
Kq = torch.randn(720, 1280, device=dev, generator=g) * 0.02
Rq = prnu.residual(Iq, zero_mean=True)
plan = prnu.PcePlan(720, 1280, 3)
plan.set_residual(Rq)
r = plan.match_template(Kq, Iq)
out["pce720_t"], out["pce720_t_peak"] = r.pce, r.peak
r = plan.match(prnu.pce_template(Kq, Iq))
out["pce720_c"] = r.peak
for (H2, W2) in ((96, 160), (45, 60)):
    I2 = u8(2, H2, W2)
    R2 = prnu.residual(I2.float(), zero_mean=True)
    r = prnu.pce(R2, prnu.pce_template(Kq[:H2, :W2].contiguous(), I2))
    out[f"pce_{H2}x{W2}"] = r.peak
Ib = u8(1, 1000, 1000)
Rb = prnu.residual(Ib, zero_mean=True)[0]
Kb = torch.randn(1000, 1000, device=dev, generator=g) * 0.02
pb, nb = prnu.block_match(Rb, prnu.pce_template(Kb, Ib)[0], 500)
out["blk500_pce"], out["blk500_ncc"] = pb, nb
out["wdft"] = prnu.wdft(torch.stack([out["fp_d3_K"], out["fp_d1_K"]]))
for taps, bnd, tr in ((16, 0, 0), (8, 1, 0), (8, 1, 1)):
    out[f"var_{taps}_{bnd}_{tr}"] = prnu.residual_variant(u8(2, 40, 52).float(), prnu.DenoiseVariant(taps, bnd, tr))
for taps, bnd in ((16, 0), (8, 1)):   # the tile kernels with interior tiles
    out[f"var_{taps}_{bnd}_0_270x480"] = prnu.residual_variant(u8(3, 270, 480).float(), prnu.DenoiseVariant(taps, bnd, 0))
torch.cuda.synchronize()
print(f"workload {time.perf_counter() - t0:.2f} s")
out = {k: t.cpu() for k, t in out.items()}
if mode == "save":
    torch.save(out, path)
    print(f"saved {len(out)} outputs")
else:
    ref = torch.load(path)
    bad = [k for k in ref if not torch.equal(ref[k], out[k])]
    print(f"compared {len(ref)} outputs: {len(bad)} differ" + (f": {bad}" if bad else " (bit-identical)"))
    sys.exit(1 if bad else 0)
