"""Opcode mix of one kernel launch from an ncu report's SASS source page."""
import csv
import re
import subprocess
import sys
from collections import defaultdict

rep, idx = sys.argv[1], sys.argv[2]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--launch-skip", idx,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Address")
ie = hdr.index("Instructions Executed")
mix = defaultdict(float)
for r in rows:
    if len(r) <= ie or not r[0].startswith("0x"):
        continue
    ins = r[1].strip()
    ins = re.sub(r"^@!?U?P\w+\s+", "", ins)
    op = ins.split()[0] if ins else "?"
    try:
        mix[op] += float(r[ie] or 0)
    except ValueError:
        pass
tot = sum(mix.values())
print(f"total warp-level instructions {tot:.0f}")
for op, v in sorted(mix.items(), key=lambda x: -x[1])[:40]:
    print(f"{op:28s} {v:14.0f} {100*v/tot:5.1f}%")
