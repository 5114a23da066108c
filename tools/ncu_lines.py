"""Per-CUDA-source-line dynamic instruction counts of one kernel (ncu source page,
cuda,sass correlation):  python tools/ncu_lines.py report.ncu-rep kernel-regex [top]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname = None
cnt = collections.Counter()
ops = collections.defaultdict(collections.Counter)
src = {}
hdr = None
T = 0
fn = None
cur = None
for r in rows:
    if len(r) >= 2 and r[0] == "Function Name":   # the first kernel only (a report can hold several)
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
    if hdr is None or len(r) != len(hdr):
        continue
    line, text, sass = r[0], r[1], r[3]
    v = r[hdr.index("Instructions Executed")]
    n = int(v) if v.isdigit() else 0
    if line.isdigit():                 # a source line: its totals
        cur = (fname, int(line))
        src[cur] = text.strip()
        cnt[cur] += n
        T += n
        continue
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", sass)
    if m and cur is not None:
        ops[cur][m.group(2)] += n
print("total", T)
for key, n in cnt.most_common(top):
    o = ", ".join(f"{k}:{v * 100 / n:.0f}%" for k, v in ops[key].most_common(4))
    print(f"{n / T * 100:5.1f}% {key[0]}:{key[1]:<5d} {src[key][:70]:70s} | {o}")
