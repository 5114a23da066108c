"""Hot SASS of one launch: executed count per instruction, with neighbours, filtered by opcode regex.
usage: ncu_sass_hot.py report launch_idx opcode_regex [n]"""
import csv, re, subprocess, sys
rep, idx, pat = sys.argv[1], sys.argv[2], sys.argv[3]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--launch-skip", idx,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = [r for r in csv.reader(txt.splitlines()) if r and r[0].startswith("0x")]
hdr = next(r for r in csv.reader(txt.splitlines()) if r and r[0] == "Address")
ie = hdr.index("Instructions Executed")
ins = [(int(r[0], 16), r[1].strip(), float(r[ie] or 0)) for r in rows]
hits = [i for i, x in enumerate(ins) if re.search(pat, x[1])]
tot = sum(ins[i][2] for i in hits)
print(f"{len(hits)} static, {tot:.0f} executed")
# group consecutive runs
for i in sorted(hits, key=lambda i: -ins[i][2])[:n]:
    a, s, c = ins[i]
    print(f"{i:6d} {c:12.0f}  {s}")
