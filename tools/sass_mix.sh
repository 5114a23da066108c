#!/bin/bash
# static SASS opcode counts of kernels whose mangled name matches $1 (in libprnu.so)
lib=${2:-/root/repo/paper_1909_04573_b200/libprnu.so}
cuobjdump -sass "$lib" 2>/dev/null | awk -v pat="$1" '/Function :/ { keep = ($0 ~ pat) } keep' |
  grep -oE "^\s+/\*[0-9a-f]{4}\*/\s+[A-Z@!][^ ;]*( [A-Z0-9_.]+)?" |
  awk '{ if ($2 ~ /^@/) print $3; else print $2 }' | sort | uniq -c | sort -rn | head -${3:-14}
