"""Per-source-line warp-stall samples (all / not-issued) of one kernel:
   python tools/ncu_stall_lines.py report.ncu-rep kernel-regex [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, res, fn, fname, tot = None, [], None, "", 0.0
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
    try:
        a = float(d.get("Warp Stall Sampling (All Samples)", "0").replace(",", "") or 0)
        n = float(d.get("Warp Stall Sampling (Not-issued Samples)", "0").replace(",", "") or 0)
    except ValueError:
        continue
    tot += a
    res.append((a, n, fname + ":" + r[0], r[1].strip()[:80]))
for a, n, ln, src in sorted(res, reverse=True)[:top]:
    print(f"{100 * a / tot:5.1f}% (not issued {100 * n / tot:4.1f}%) {ln:>16s}  {src}")
