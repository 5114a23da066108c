"""Per-source-line shared-memory wavefronts (total / excessive) and instructions of one
kernel:  python tools/ncu_smem_lines.py report.ncu-rep kernel-regex [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, res, fn, fname = None, [], None, ""
for r in rows:
    if len(r) >= 2 and r[0] == "Function Name":
        if fn is not None and r[1] != fn:
            break
        fn = r[1]
        continue
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or not r[0].isdigit():
        continue
    d = dict(zip(hdr, r))

    def f(k):
        try:
            return float(d.get(k, "0").replace(",", ""))
        except ValueError:
            return 0.0
    res.append((f("L1 Wavefronts Shared"), f("L1 Wavefronts Shared Excessive"), f("Instructions Executed"),
                fname + ":" + r[0],
                r[1].strip()[:72]))
for wf, ex, ins, ln, src in sorted(res, reverse=True)[:top]:
    print(f"{ln:>16s} wf {wf / 1e6:7.2f}M ex {ex / 1e6:6.2f}M inst {ins / 1e6:6.2f}M  {src}")
