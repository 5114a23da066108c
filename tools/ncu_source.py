"""Per-CUDA-source-line aggregation of an ncu report's source page (needs -lineinfo).
usage: ncu_source.py report.ncu-rep launch_index [top]"""
import csv
import subprocess
import sys

rep, idx = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda", "--launch-skip", idx,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
print(rows[0][:2])
hdr = rows[1]
ci = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    def f(k):
        try:
            return float(r[ci[k]]) if k in ci and r[ci[k]] not in ("", "-") else 0.0
        except ValueError:
            return 0.0
    data.append((r[ci["Line"]] if "Line" in ci else r[0], r[ci["Source"]][:90], f("Warp Stall Sampling (All Samples)"),
                 f("L1 Wavefronts Shared"), f("L1 Wavefronts Shared Ideal"), f("Instructions Executed")))
tot_s = sum(d[2] for d in data) or 1
tot_w = sum(d[3] for d in data) or 1
tot_i = sum(d[5] for d in data) or 1
print(f"total samples {tot_s:.0f} shared wavefronts {tot_w:.0f} (ideal {sum(d[4] for d in data):.0f}) inst {tot_i:.0f}")
for d in sorted(data, key=lambda x: -x[2])[:top]:
    print(f"{d[0]:>5} stall {100*d[2]/tot_s:5.1f}%  wf {100*d[3]/tot_w:5.1f}% (ideal {d[4]:.0f}/{d[3]:.0f})  inst {100*d[5]/tot_i:5.1f}%  {d[1]}")
