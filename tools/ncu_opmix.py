"""Dynamic SASS opcode mix of one kernel from an ncu report (source page):
   python tools/ncu_opmix.py report.ncu-rep [kernel-regex] [positions]
Prints warp-instructions per opcode (and per position if given) with shared-memory
wavefronts and stall samples."""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else None
npos = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if kern:
    cmd += ["-k", "regex:" + kern]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if "Source" in r and "Instructions Executed" in r)
i0 = rows.index(hdr)
data = []
for r in rows[i0 + 1:]:   # the first kernel's section only (a report can hold several)
    if len(r) == len(hdr) and r[0] == hdr[0]:
        break
    if len(r) == len(hdr):
        data.append(r)
iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
iW, iSm = hdr.index("L1 Wavefronts Shared"), hdr.index("Warp Stall Sampling (All Samples)")
tot, wf, st = collections.Counter(), collections.Counter(), collections.Counter()
T = 0
for r in data:
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.\S+)?", r[iS])
    if not m:
        continue
    op = m.group(2)
    key = op + (m.group(3) or "") if op in ("LDS", "STS", "LDG", "STG") else op
    n = int(r[iE]) if r[iE].isdigit() else 0
    T += n
    tot[key] += n
    wf[key] += int(r[iW]) if r[iW].isdigit() else 0
    st[key] += int(r[iSm]) if r[iSm].isdigit() else 0
print(f"total warp-instructions {T}" + (f"  per position (thread-instr) {T * 32 / npos:.1f}" if npos else ""))
for k, v in tot.most_common(45):
    per = f" {v * 32 / npos:7.2f}/pos" if npos else ""
    print(f"{k:16s} {v:12d} {v / T * 100:5.1f}%{per}  wf {wf[k]:10d}  stall {st[k]}")
