"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per-kernel
launches, total time and share, for this library's kernels (namespace prnu::)."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
hdr = rows[0]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = defaultdict(float)
cnt = defaultdict(int)
other = 0.0
for r in rows[1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
    name = r[ki]
    if not any(t in name for t in ("prnu::", "splitk::", "fft::k_pce")):   # ncu prints prnu::fft:: as fft::
        other += v * scale
        continue
    short = name.split("(")[0].replace("void ", "").replace("prnu::", "").replace("splitk::", "").replace("fft::", "")
    tot[short] += v * scale
    cnt[short] += 1
T = sum(tot.values())
print(f"{'kernel':45s} {'launches':>8s} {'total us':>10s} {'avg us':>9s} {'share':>6s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:45s} {cnt[k]:8d} {tot[k]:10.1f} {tot[k]/cnt[k]:9.2f} {100*tot[k]/T:5.1f}%")
print(f"prnu kernels total {T:.1f} us; non-prnu (torch input generation, cuFFT) {other:.1f} us")
