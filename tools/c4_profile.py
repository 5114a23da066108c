"""Camera-identification workload (BASELINE config 4) split: fingerprints vs PCE matrix."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_04573_b200 as prnu
import synth

H, W, n = 720, 1280, 64
fr = synth.video("drift", 301, H, W, seed=4, camera=0, device="cuda").frames
ex = prnu.Extractor(H, W, 30, 10)
Iq = fr[300:301].expand(n, H, W).contiguous()
plan = prnu.PcePlan(H, W, n)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


Ks = [ex(fr[:300]).K.clone() for _ in range(n)]
nst = 8
exs = [prnu.Extractor(H, W, 30, 10) for _ in range(nst)]
sts = [torch.cuda.Stream() for _ in range(nst)]
Kout = torch.empty((n, H, W), device="cuda")


def fps_streams():
    cur = torch.cuda.current_stream()
    for s_ in sts:
        s_.wait_stream(cur)
    for c in range(n):
        with torch.cuda.stream(sts[c % nst]):
            Kout[c].copy_(exs[c % nst](fr[:300]).K)
    for s_ in sts:
        cur.wait_stream(s_)


print("64 fingerprints on 8 streams %.2f ms" % timed(fps_streams))
R = prnu.residual(Iq, zero_mean=True)
print("64 fingerprints  %.2f ms" % timed(lambda: [ex(fr[:300]) for _ in range(n)]))
print("64 query residuals %.2f ms" % timed(lambda: prnu.residual(Iq, zero_mean=True)))
print("64x64 templates  %.2f ms" % timed(lambda: [prnu.pce_template(Ks[c], Iq) for c in range(n)]))
T = prnu.pce_template(Ks[0], Iq)
print("64x64 PCE        %.2f ms" % timed(lambda: [plan(R, T) for c in range(n)]))
plan.set_residual(R)
print("64x64 PCE cached %.2f ms" % timed(lambda: [plan.match(T) for c in range(n)]))
print("64x64 PCE cached, fused templates %.2f ms" % timed(lambda: [plan.match_template(Ks[c], Iq) for c in range(n)]))
prnu._lib.prnu_profile_begin()
plan(R, T)
torch.cuda.synchronize()
import ctypes
maxk = 32
names = ctypes.create_string_buffer(64 * maxk)
tot = (ctypes.c_double * maxk)()
cnt = (ctypes.c_int64 * maxk)()
nk = ctypes.c_int()
prnu._lib.prnu_profile_end(maxk, names, tot, cnt, ctypes.byref(nk))
for k in range(nk.value):
    print("   ", names.raw[64 * k: 64 * k + 64].split(b"\0")[0].decode(), "%.3f ms" % tot[k], cnt[k])

# concurrent plans: cameras dealt over streams, one plan (and cached residual spectrum) per stream
for nst in (2, 3, 4):
    plans = [prnu.PcePlan(H, W, n) for _ in range(nst)]
    for p_ in plans:
        p_.set_residual(R)
    streams = [torch.cuda.Stream() for _ in range(nst)]

    def multi():
        cur = torch.cuda.current_stream()
        for s_ in streams:
            s_.wait_stream(cur)
        for c in range(n):
            with torch.cuda.stream(streams[c % nst]):
                plans[c % nst].match_template(Ks[c], Iq)
        for s_ in streams:
            cur.wait_stream(s_)
    print("64x64 PCE cached, fused templates, %d streams %.2f ms" % (nst, timed(multi)))
    del plans
