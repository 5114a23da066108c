"""Per-CUDA-source-line aggregation of one kernel launch in an ncu report (needs -lineinfo).
usage: ncu_source.py report.ncu-rep launch_index [top]"""
import csv
import subprocess
import sys

rep, idx = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--launch-skip",
                      idx, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
cur_file, hdr, data = "", None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        print(r[1])
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    ci = {h: i for i, h in enumerate(hdr) if h not in ("Source",) or i == 1}

    def f(k):
        i = hdr.index(k) if k in hdr else -1
        try:
            return float(r[i]) if i >= 0 and r[i] not in ("", "-") else 0.0
        except ValueError:
            return 0.0
    data.append((f"{cur_file}:{r[0]}", r[1][:80], f("Warp Stall Sampling (All Samples)"), f("L1 Wavefronts Shared"),
                 f("L1 Wavefronts Shared Ideal"), f("Instructions Executed")))
tot_s = sum(d[2] for d in data) or 1
tot_w = sum(d[3] for d in data) or 1
tot_i = sum(d[5] for d in data) or 1
print(f"samples {tot_s:.0f}  shared wavefronts {tot_w:.0f} (ideal {sum(d[4] for d in data):.0f})  inst {tot_i:.0f}")
for d in sorted(data, key=lambda x: -x[2])[:top]:
    print(f"{d[0]:>16} stall {100*d[2]/tot_s:5.1f}%  wf {100*d[3]/tot_w:5.1f}% ({d[3]:.0f}/ideal {d[4]:.0f})"
          f"  inst {100*d[5]/tot_i:5.1f}%  {d[1]}")
