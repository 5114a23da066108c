#!/bin/bash
# ncu --set full of ONE launch of a kernel (base-name regex) during tools/profile_extract.py,
# then print every raw metric whose name matches a grep pattern.
# usage: tools/ncu_raw_grep.sh [kernel-regex] [pattern] [out-name]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
K=${1:-k_analysis_lift}; PAT=${2:-wavefronts|sectors|requests}; OUT=${3:-gpurun_out/rawcap}
python tools/profile_extract.py 64 64 > /dev/null 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$K" --launch-skip ${SKIP:-0} -c 1 -f -o $OUT \
  python tools/profile_extract.py 64 64 > gpurun_out/ncu_raw.log 2>&1
echo "ncu rc $?"; tail -2 gpurun_out/ncu_raw.log
ncu -i $OUT.ncu-rep --page raw --csv > $OUT.raw.csv
python - "$OUT.raw.csv" "$PAT" <<'EOF'
import csv, re, sys
r = list(csv.reader(open(sys.argv[1])))
hdr, units = r[0], r[1]
pat = re.compile(sys.argv[2])
for row in r[2:]:
    print(row[hdr.index('Kernel Name')][:60])
    for i, h in enumerate(hdr):
        if pat.search(h) and row[i] not in ('', '0', 'n/a'):
            print(f"   {h:80s} {units[i]:10s} {row[i]}")
EOF
