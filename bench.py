#!/usr/bin/env python
"""bench.py — SDA-frame PRNU fingerprint extraction on B200 (BASELINE config 2).

One step = the whole hot path over one synthetic 1800-frame
1920x1080 u8 video resident in HBM:
  * conventional fingerprint (depth 1: 1800 denoisings)            a2-a6
  * SDA fingerprint (depth 50: averaging + 36 denoisings)          a1-a6
  * NCC of both fingerprints against the true K                    a7
  * residual of a fresh query frame + PCE vs both fingerprints     a2-a4, a8
metric: denoised Full-HD frames/s (1836 fingerprint denoisings per step), with
fingerprints/s per depth beside it.  `e2e` repeats the two extractions through
the host-buffer C-ABI call (frames in pinned host memory, K back to the host).

python bench.py [--gpus N --steps K --warmup W] [--impl reference]
N > 1 runs N independent replicas (one video per rank; DESIGN.md "replicas
only"), launched by torchrun; timing is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import re
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["prnu", "reference"], default="prnu")
    ap.add_argument("--frames", type=int, default=1800)
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--width", type=int, default=1920)
    ap.add_argument("--depths", default="1,50")
    ap.add_argument("--batch", type=int, default=0,
                    help="SDA frames denoised per wave at depth 1 (0: waves of <= 360 frames, equal sizes)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--e2e-batch", type=int, default=64, help="frames per upload chunk / wave of the e2e run")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the NEXT-row measurements (f1, f2, f4)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="budget of the oracle sample")
    ap.add_argument("--serial-depths", action="store_true", help="run the depths one after the other (A/B)")
    return ap.parse_args()


# ------------------------------------------------------------------ dist
def dist_setup(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if torch.cuda.is_available() and dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# BASELINE.json's metric; `value` is its first quantity (denoised Full-HD frames/s),
# fingerprints/s and the HBM fraction are reported beside it.
BASELINE_METRIC = "denoised Full-HD frames/sec and fingerprints/sec (1800-frame video) at 1 B200; % HBM peak"


def job_throughput(units_per_step: float, steps: int, world: int, ms_max: float) -> float:
    """Whole-job throughput: units every rank processed / the slowest rank's time."""
    return units_per_step * steps * world / (ms_max / 1000.0)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clock + throttle reasons with NVML every 20 ms while active."""

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                 "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4, "applications_clocks_setting": 0x2}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s)}


# ------------------------------------------------------------------ roofline model
def sub_len(n):
    return (n + 7) // 2


# FP32-pipe lane-operations per level-l coefficient position of the lifted analysis
# (DESIGN.md §6): the lifting DWT costs 8 FMA per (a, d) pair -> rows 2 x 8 + columns
# 2 x 8 = 32, + 1 (the LL scale); the shrink of 3 detail coefficients, each c^2 (1) +
# nested vertical (8) + sliding horizontal (8) window sums + 4 scalings + the Wiener
# product (2) = 23 -> 69.  min / max / rcp run on other pipes (not counted).
ALU_OPS_PER_POSITION = 33 + 3 * 23
FP32_LANES_PER_SM = 128


def algorithmic_ops_per_step(name: str, H: int, W: int, levels: int, depths, m: int, n_query: int = 1):
    """FP32 lane-ops one step needs in an analysis kernel (fused DWT + shrink) of `name`."""
    if not name.startswith("analysis_l"):
        return None
    l = int(name[len("analysis_l")])
    nH, nW = H, W
    for _ in range(l):
        nH, nW = sub_len(nH), sub_len(nW)
    f_u8 = (m if 1 in depths else 0) + n_query
    f_pair = sum(m // d for d in depths if d == 2)
    f_u16 = sum(m // d for d in depths if 2 < d <= 257)
    f_f32 = sum(m // d for d in depths if d > 257)
    frames = {"_u8": f_u8, "u16": f_u16, "f32": f_f32, "air": f_pair}.get(name[-3:], f_u8 + f_pair + f_u16 + f_f32)
    return frames * nH * nW * ALU_OPS_PER_POSITION


def algorithmic_bytes_per_step(name: str, H: int, W: int, levels: int, depths, m: int, n_query: int = 1):
    """Algorithmic HBM bytes one step moves through kernel `name`:
    each input read once and each output written once at real (unpadded) sizes;
    NUM/DEN (fp64) read + written once per synth_acc launch (counted by caller).
    Frames per step: depth-1 fingerprint m (u8 input), SDA fingerprints m//d
    (fp32 input), query residual n_query (u8 input)."""
    nH, nW = [H], [W]
    for _ in range(levels):
        nH.append(sub_len(nH[-1]))
        nW.append(sub_len(nW[-1]))
    n = [nH[l] * nW[l] for l in range(levels + 1)]
    P = H * W
    f_u8 = (m if 1 in depths else 0) + n_query                 # level-1 u8 inputs
    f_pair = sum(m // d for d in depths if d == 2)             # SDA pairs: both u8 frames staged by the kernels
    f_u16 = sum(m // d for d in depths if 2 < d <= 257)        # SDA frames as exact u16 group sums
    f_f32 = sum(m // d for d in depths if d > 257)             # SDA frames as fp32
    f_all = f_u8 + f_pair + f_u16 + f_f32
    if name == "sda_sum":                                       # d u8 frames read, u16 sum written
        return sum((m // d) * (d * P + 2 * P) for d in depths if 2 < d <= 257)
    if name == "sda_average":
        return sum((m // d) * (d * P + 4 * P) for d in depths if d > 257)
    if name == "analysis_l1_u8":
        return f_u8 * (1 * P + 4 * 4 * n[1])
    if name == "analysis_l1_u16":
        return f_u16 * (2 * P + 4 * 4 * n[1])
    if name == "analysis_l1_pair":
        return f_pair * (2 * P + 4 * 4 * n[1])
    if name == "analysis_l1_f32":
        return f_f32 * (4 * P + 4 * 4 * n[1])
    lvl = re.match(r"(analysis|synthesis)_l(\d)$", name)
    if lvl and lvl.group(1) == "analysis":
        l = int(lvl.group(2))
        return f_all * (4 * n[l - 1] + (4 if l < levels else 3) * 4 * n[l])
    if lvl and lvl.group(1) == "synthesis" and name != "synthesis_l1":
        l = int(lvl.group(2))
        return f_all * ((4 if l < levels else 3) * 4 * n[l] + 4 * n[l - 1])
    if name == "synthesis_l1":
        return n_query * (4 * 4 * n[1] + 4 * P)
    if name == "synth_acc_l1_u8":
        return (m if 1 in depths else 0) * (4 * 4 * n[1] + 1 * P)
    if name == "synth_acc_l1_u16":
        return f_u16 * (4 * 4 * n[1] + 2 * P)
    if name == "synth_acc_l1_pair":
        return f_pair * (4 * 4 * n[1] + 2 * P)
    if name == "synth_acc_l1_f32":
        return f_f32 * (4 * 4 * n[1] + 4 * P)
    return None


def sda_batch(n: int) -> int:
    """SDA frames per wave: equal waves of at most 360 (as the depth-1 default)."""
    nw = -(-n // 360)
    return max(1, -(-n // nw))


# ------------------------------------------------------------------ reference arm / cpu baseline
def run_reference(args, rank, world):
    """--impl reference: the fp64 CPU oracle on the host cores (rank 0 only)."""
    import numpy as np
    import torch

    import synth
    if rank != 0:
        return
    depths = [int(x) for x in args.depths.split(",")]
    m = min(args.frames, max(depths) * 2)
    v = synth.video("drift", m, args.height, args.width, seed=0,
                    device="cuda" if torch.cuda.is_available() else "cpu")
    fr = v.frames.cpu().numpy()
    from oracle import parallel
    per_step = max(2.0, min(args.cpu_seconds * 4, 120.0) / max(1, args.steps + args.warmup))
    for _ in range(args.warmup):
        parallel.sample(fr, depths, per_step)
    rates = []
    t_all = 0.0
    desc, nproc = "", 1
    for _ in range(args.steps):
        t0 = time.perf_counter()
        r, nproc, desc = parallel.sample(fr, depths, per_step)
        t_all += time.perf_counter() - t0
        rates.append(r)
    value = float(np.mean(rates))
    line = {"impl": "reference", "metric": BASELINE_METRIC, "value": value,
            "unit": "denoised FHD frames/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * t_all / max(1, args.steps), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded Eq. 1 sensor model, DESIGN.md §4)",
            "config": {"workload": f"C2 {args.frames}x{args.height}x{args.width} u8 video, depths {depths} "
                                   "(bounded oracle sample per step)",
                       "frames": args.frames, "H": args.height, "W": args.width, "depths": depths},
            "cpu_baseline": {"value": value, "unit": "denoised FHD frames/s", "cores": nproc, "kind": "oracle",
                             "sample": f"{nproc} worker processes (one per host core), last step: {desc}"},
            "e2e": {"value": value, "unit": "denoised FHD frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ main arm
def variant_alg_bytes(H, W, levels, taps, boundary, transform):
    """Algorithmic HBM bytes of one f3 variant residual (csrc/variant.cu), fp32: decimated
    variants (fused tile kernels) read each level's input and write its four subbands once,
    the shrink reads and writes three planes, each synthesis level reads four (three at the
    coarsest) subbands and writes its output; undecimated variants (separable passes) also
    move the row-pass intermediates."""
    m = 1 << levels
    h, w = H, W
    tot = 0
    dims = []
    for l in range(1, levels + 1):
        ph = (h + m - 1) // m * m if (boundary and not transform and l == 1) else h
        pw = (w + m - 1) // m * m if (boundary and not transform and l == 1) else w
        if transform:
            nh, nw = h, w
        elif boundary:
            nh, nw = ph // 2, pw // 2
        else:
            nh, nw = (h + taps - 1) // 2, (w + taps - 1) // 2
        dims.append((h, w, nh, nw))
        tot += h * w + 4 * nh * nw           # analysis in, four subbands out
        if transform:
            tot += 4 * h * nw                # row-pass intermediates (lo, hi) written + read
        tot += 6 * nh * nw                   # shrink (3 in, 3 out)
        h, w = nh, nw
    for l in range(levels, 0, -1):
        ih, iw, nh, nw = dims[l - 1]
        tot += (3 if l == levels else 4) * nh * nw + ih * iw       # synthesis in / out
        if transform:
            tot += 4 * ih * nw                                     # column-pass intermediates
    return 4 * tot


def main():
    args = parse()
    rank, world, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import numpy as np
    import torch

    import paper_1909_04573_b200 as prnu
    import synth

    assert torch.cuda.is_available(), "bench.py needs a CUDA device"
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    depths = [int(x) for x in args.depths.split(",")]
    m, H, W = args.frames, args.height, args.width

    # ---- inputs: one synthetic video per rank (+1 query frame), resident in HBM
    allf = torch.empty((m + 1, H, W), dtype=torch.uint8, device=dev)
    v = synth.video("drift", m + 1, H, W, seed=rank, device=dev, out=allf)
    frames, query = allf[:m], allf[m:]
    K_true = v.K.contiguous()
    torch.cuda.synchronize()

    if args.batch <= 0:   # equal waves of at most 360 frames (1800 -> 5 waves of 360; measured best)
        nw = -(-m // 360)
        args.batch = -(-m // nw)
    exs = {d: prnu.Extractor(H, W, d, batch=(args.batch if d == 1 else sda_batch(m // d)), device=dev)
           for d in depths}
    n_sda = {d: m // d for d in depths}
    plan = prnu.PcePlan(H, W, len(depths), device=dev)

    side = torch.cuda.Stream(device=dev)                # least priority: fills the gaps
    main_hp = torch.cuda.Stream(device=dev, priority=-1)   # depth 1 (the library's wave streams inherit it)

    def step(concurrent=True):
        # The depths are independent fingerprints of the same frames, and the query residual
        # needs none of them: the first depth runs on the current stream, the query residual
        # and the other depths on a side stream (the SDA group sums are HBM-bound, the
        # depth-1 denoising L1-bound, the one-frame residual latency-bound: they overlap);
        # the per-kernel timing pass runs everything in order so each kernel is timed alone.
        Ks = [None] * len(depths)
        cur = torch.cuda.current_stream()
        if concurrent and not args.serial_depths:
            side.wait_stream(cur)   # also: the previous step's readers of the side outputs are done
            main_hp.wait_stream(cur)
            with torch.cuda.stream(side):
                Rq = prnu.residual(query, zero_mean=True)
                for k in range(1, len(depths)):
                    Ks[k] = exs[depths[k]](frames).K
            with torch.cuda.stream(main_hp):
                Ks[0] = exs[depths[0]](frames).K
            cur.wait_stream(main_hp)
            cur.wait_stream(side)
        else:
            for k, d in enumerate(depths):
                Ks[k] = exs[d](frames).K
            Rq = prnu.residual(query, zero_mean=True)
        for K in Ks:
            prnu.ncc(K, K_true)
        T = prnu.pce_template(torch.stack(Ks), query.expand(len(depths), H, W).contiguous())
        return plan(Rq.expand(len(depths), H, W).contiguous(), T)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = prnu.kernel_launches()
    sampler = ClockSampler(dev.index)
    barrier(world)
    torch.cuda.synchronize()
    with sampler:
        e0.record(stream)
        for _ in range(args.steps):
            res = step()
        e1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    ms = e0.elapsed_time(e1)
    launches = prnu.kernel_launches() - launches0
    ms_max = max_over_ranks(ms, world)
    ms_step = ms_max / args.steps
    denoise_per_step = sum(n_sda.values())
    value = job_throughput(denoise_per_step, args.steps, world, ms_max)
    pce_vals = res.pce.cpu().tolist()

    # ---- per-kernel event timing over the same K steps (separate pass; the
    #      library serialises its waves while timing so each kernel is measured alone)
    roof, kernels = None, None
    if not args.no_profile:
        prnu._lib.prnu_profile_begin()
        for _ in range(args.steps):
            step(concurrent=False)
        torch.cuda.synchronize()
        import ctypes
        maxk = 64
        names = ctypes.create_string_buffer(64 * maxk)
        tot = (ctypes.c_double * maxk)()
        cnt = (ctypes.c_int64 * maxk)()
        nk = ctypes.c_int()
        prnu._lib.prnu_profile_end(maxk, names, tot, cnt, ctypes.byref(nk))
        kernels = {}
        for k in range(min(nk.value, maxk)):
            nm = names.raw[64 * k: 64 * k + 64].split(b"\0")[0].decode()
            kernels[nm] = {"ms_per_step": tot[k] / args.steps, "launches_per_step": cnt[k] / args.steps}
        tot_ms = sum(x["ms_per_step"] for x in kernels.values())
        peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
        peaks = json.load(open(peaks_path)) if os.path.exists(peaks_path) else {}
        peak = peaks.get("hbm_gbs", 6650.0)
        for nm, x in kernels.items():
            x["share"] = x["ms_per_step"] / tot_ms
            by = algorithmic_bytes_per_step(nm, H, W, 4, depths, m)
            if by is not None and nm.startswith("synth_acc"):
                by += 32 * H * W * x["launches_per_step"]          # NUM/DEN read + write per launch
            if by is not None:
                x["alg_bytes_per_launch"] = by / x["launches_per_step"]
                x["alg_GBps"] = by / (x["ms_per_step"] / 1000.0) / 1e9
                x["frac_hbm"] = x["alg_GBps"] / peak
        # dominant kernel = largest share of kernel time
        top = max(kernels, key=lambda k: kernels[k]["ms_per_step"])
        kt = kernels[top]
        avg_ms = kt["ms_per_step"] / kt["launches_per_step"]
        achieved = kt.get("alg_GBps")
        # DRAM traffic per launch of that kernel from the committed ncu --set full capture
        # (same kernel and launch configuration), else null
        # (bytes per frame of the capture x this run's average frames per launch)
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "latest_traffic.json")
        if os.path.exists(tpath):
            t = json.load(open(tpath))
            fpl = (n_sda.get(1, 0) + 1) / max(1.0, kt["launches_per_step"]) if top.endswith("_u8") else None
            if t.get("kernel") == top and fpl and t.get("H") == H and t.get("W") == W:
                traffic = (t["dram_bytes_read"] + t["dram_bytes_write"]) / t["frames_per_launch"] * fpl
        hbm_view = {"achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                    "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback",
                    "bytes_per_launch": kt.get("alg_bytes_per_launch")}
        ops = algorithmic_ops_per_step(top, H, W, 4, depths, m)
        # BASELINE.json asks for the HBM fraction of the denoise / accumulate kernels: the
        # line's roofline is the HBM one.  The fused analysis is bound by FP32 issue, not by
        # HBM, so its FP32-pipe roofline is reported beside it: algorithmic
        # lane-ops / launch time vs 148 SMs x 128 lanes x the max SM clock.
        roof = dict(kernel=top, bound="hbm", avg_launch_ms=avg_ms, share_of_kernel_time=kt["share"], **hbm_view)
        if ops is not None:
            sm_mhz = peaks.get("sm_max_mhz", 1965.0)
            n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
            alu_peak = n_sm * FP32_LANES_PER_SM * sm_mhz * 1e6 / 1e12
            alu_ach = ops / (kt["ms_per_step"] / 1000.0) / 1e12
            roof["alu_view"] = {"bound_note": "bound by the L1/shared-memory data pipe and issue, not HBM "
                                              "(DESIGN.md §6)",
                                "achieved": alu_ach, "peak": alu_peak, "unit": "T fp32 lane-op/s",
                                "frac": alu_ach / alu_peak, "ops_per_launch": ops / kt["launches_per_step"],
                                "peak_source": "derived: %d SM x 128 FP32 lanes x %.0f MHz" % (n_sm, sm_mhz)}

    # ---- NEXT rows, measured outside the step: f2 WDFT of the two
    #      fingerprints, f1 500x500 block matching of the query, f4 RGB->luma
    next_rows = None
    if not args.no_extras and rank == 0:   # measured outside the step, reported by rank 0 only
        def timed(fn, reps=5):
            fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(torch.cuda.current_stream())
            for _ in range(reps):
                fn()
            b.record(torch.cuda.current_stream())
            torch.cuda.synchronize()
            return a.elapsed_time(b) / reps
        Ks2 = torch.stack([exs[d](frames).K for d in depths])
        wplan = prnu.WdftPlan(H, W, len(depths), device=dev)
        t_wdft = timed(lambda: wplan(Ks2))
        Rq = prnu.residual(query, zero_mean=True)[0]
        Tq = prnu.pce_template(Ks2[0], query)[0]
        bplan = prnu.BlockPlan(H, W, 500, device=dev)
        t_blk = timed(lambda: bplan(Rq, Tq))
        rgb = torch.randint(0, 256, (16, 3, H, W), dtype=torch.uint8, device=dev)
        t_luma = timed(lambda: prnu.rgb_to_luma(rgb))
        luma_bytes = 16 * H * W * (3 + 4)
        pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
        peak_hbm = json.load(open(pk)).get("hbm_gbs", 6650.0) if os.path.exists(pk) else 6650.0
        # f3 denoiser variants: residual of 64 FHD SDA-like fp32 frames per call
        Ivar = frames[:64].float()
        f3 = {}
        # the default denoiser (db4, symmetric) through the same residual call on the same fp32
        # frames: the like-for-like denominator (x_default divides by the fused u8 extraction's
        # per-denoise time, which reads 1 B/px and writes no residual)
        out_def = torch.empty_like(Ivar)
        t_def = timed(lambda: prnu.residual(Ivar, out=out_def), reps=3)
        f3["db4_sym_default"] = {"ms_per_frame": t_def / Ivar.shape[0],
                                 "x_default": (t_def / Ivar.shape[0]) / (ms_step / denoise_per_step)}
        for name, v in (("db8_sym", (16, 0, 0)), ("db4_per", (8, 1, 0)), ("db8_per", (16, 1, 0)),
                        ("db4_swt", (8, 1, 1)), ("db8_swt", (16, 1, 1))):
            var = prnu.DenoiseVariant(*v)
            out = torch.empty_like(Ivar)
            t = timed(lambda: prnu.residual_variant(Ivar, var, out=out), reps=3)
            gb = variant_alg_bytes(H, W, 4, *v) * Ivar.shape[0] / (t / 1000.0) / 1e9
            f3[name] = {"ms_per_frame": t / Ivar.shape[0], "alg_GBps": gb, "frac_hbm": gb / peak_hbm,
                        "x_default": (t / Ivar.shape[0]) / (ms_step / denoise_per_step),
                        "x_default_residual": t / t_def}
        # BASELINE config 4 shape (camera identification): 64 fingerprints of 300 frames
        # 1280x720 at depth 30, then 64 query residuals x 64 fingerprints = 4096 PCEs
        # (one camera's synthetic frames reused for every camera: throughput only)
        c4H, c4W, c4n = 720, 1280, 64
        fr4 = synth.video("drift", 301, c4H, c4W, seed=4, camera=0, device=dev).frames
        ex4 = prnu.CameraBatchExtractor(c4H, c4W, 30, 10, streams=8, device=dev)
        Iq4 = fr4[300:301].expand(c4n, c4H, c4W).contiguous()
        pm4 = prnu.PceMatrix(c4H, c4W, c4n, streams=4, device=dev)

        def camera_id():
            Ks4 = ex4([fr4[:300]] * c4n)
            R4 = prnu.residual(Iq4, zero_mean=True)
            pm4.set_queries(R4, Iq4)   # one FFT of the 64 query residuals per stream plan
            pm4(Ks4)                   # 64 x 64 PCEs, templates K (.) Iq formed inside the row FFT
        t_c4 = timed(camera_id, reps=1)
        c4 = {"workload": "64 x 300 frames 1280x720, depth 30, 64x64 PCE", "ms": t_c4,
              "fingerprints_per_s": c4n / (t_c4 / 1000.0), "pce_per_s": c4n * c4n / (t_c4 / 1000.0)}
        # BASELINE config 5: one 1920x1080 stack of 3600 frames ("shift" model), depths
        # 1 .. 3600: per depth the fingerprint time, denoised frames/s, % HBM (SDA read +
        # denoise traffic) and NCC against the true K
        del fr4, Iq4, pm4, ex4
        torch.cuda.empty_cache()
        v5 = synth.video("shift", 3600, H, W, seed=5, device=dev)
        c5 = {}
        for d5 in (1, 2, 5, 10, 25, 50, 100, 300, 3600):
            ex5 = prnu.Extractor(H, W, d5, 225 if d5 == 1 else sda_batch(3600 // d5), device=dev)
            t5 = timed(lambda: ex5(v5.frames), reps=1)
            n5 = 3600 // d5
            rho = float(prnu.ncc(ex5(v5.frames).K, v5.K))
            c5[str(d5)] = {"ms": t5, "denoisings": n5, "denoised_frames_per_s": n5 / (t5 / 1000.0),
                           "source_frames_per_s": 3600 / (t5 / 1000.0), "ncc_vs_true_K": rho}
            del ex5
        del v5
        torch.cuda.empty_cache()
        # BASELINE config 3: 200 luma stills 4000x3000, depths 1, 5, 10, 20, 50
        Y3, K3 = synth.stills(200, 3000, 4000, seed=0, device=dev)
        c3 = {}
        for d3 in (1, 5, 10, 20, 50):
            ex3 = prnu.Extractor(3000, 4000, d3, 40 if d3 == 1 else max(1, 200 // d3), device=dev)
            t3 = timed(lambda: ex3(Y3), reps=1)
            n3 = 200 // d3
            c3[str(d3)] = {"ms": t3, "denoisings": n3, "denoised_Mpx_per_s": n3 * 12.0 / (t3 / 1000.0),
                           "ncc_vs_true_K": float(prnu.ncc(ex3(Y3).K, K3))}
            del ex3
        del Y3, K3
        torch.cuda.empty_cache()
        next_rows = {"f3_variants": f3, "c4_camera_id": c4, "c5_depth_sweep": c5, "c3_stills": c3,
                     "f2_wdft_ms_per_fingerprint": t_wdft / len(depths),
                     "f1_block_match_ms": t_blk, "f1_tiles": bplan.n_tiles,
                     "f4_rgb_to_luma_GBps": luma_bytes / (t_luma / 1000.0) / 1e9,
                     "f4_rgb_to_luma_frac_hbm": luma_bytes / (t_luma / 1000.0) / 1e9 / peak_hbm}

    # ---- e2e through the host-buffer C-ABI call: the frames start in pinned host
    #      memory; one upload per step feeds every depth (prnu_extract_multi_host),
    #      the fingerprints come back to host memory
    e2e = None
    if not args.no_e2e:
        host = torch.empty((m, H, W), dtype=torch.uint8, pin_memory=True)
        host.copy_(frames)
        # upload chunks = waves: smaller waves than the device-resident step's overlap the
        # PCIe stream better (the first chunk's copy is not hidden)
        mx = prnu.MultiExtractor(m, H, W, depths, batch=args.e2e_batch, device=dev)
        mx(host)
        torch.cuda.synchronize()
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            mx(host)
        t = time.perf_counter() - t0
        t = max_over_ranks(t, world)
        e2e = {"value": denoise_per_step * args.e2e_steps * world / t, "unit": "denoised FHD frames/s",
               "h2d_bytes_per_step": int(m * H * W), "d2h_bytes_per_step": int(len(depths) * H * W * 4),
               "steps": args.e2e_steps, "fingerprints_per_s": len(depths) * args.e2e_steps * world / t,
               "api": "prnu_extract_multi_host (one upload per step for all depths)"}
        del host, mx

    # ---- cpu baseline: the oracle on a bounded sample (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        fr = frames[: max(depths) * 2].cpu().numpy()   # 100 frames: 100 (d=1) / 2 (d=50) SDA groups
        from oracle import parallel
        r, nproc, desc = parallel.sample(fr, depths, args.cpu_seconds)
        cpu = {"value": r, "unit": "denoised FHD frames/s", "cores": nproc, "kind": "oracle",
               "sample": f"fp64 C oracle as it stands, {nproc} worker processes (one per host core), SDA groups "
                         f"of the first frames of the same video: {desc}"}

    if rank == 0:
        ncc_vals = [prnu.ncc(exs[d](frames).K, K_true).item() for d in depths]
        line = {
            "metric": BASELINE_METRIC,
            "value": value, "unit": "denoised FHD frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded Eq. 1 sensor model, DESIGN.md §4)",
            "config": {"workload": f"C2: {m}x{W}x{H} u8 video, fingerprints at depths {depths}, NCC vs true K, "
                                   "query residual + PCE", "frames": m, "H": H, "W": W, "depths": depths,
                       "batch": args.batch, "denoises_per_step": denoise_per_step,
                       "l2": f"inputs ({m * H * W / 1e9:.2f} GB u8) larger than the 126 MB L2; no flush",
                       "parallelism": f"replicas x{world}"},
            "fingerprints_per_s": {f"depth{d}": 1000.0 / ms_step * world for d in depths},
            "source_frames_per_s": len(depths) * m * world * 1000.0 / ms_step,
            "ncc_vs_true_K": dict(zip([f"depth{d}" for d in depths], ncc_vals)),
            "pce_query": pce_vals,
            "gpu_launches": int(launches),
            "clocks": sampler.summary(),
            "roofline": roof,
            "kernels": kernels,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "next_rows": next_rows,
        }
        print(json.dumps(line), flush=True)
    barrier(world)


if __name__ == "__main__":
    main()
