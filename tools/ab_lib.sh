#!/bin/bash
# A/B of two prebuilt libprnu.so files (A = in-tree build, B = $1), interleaved, R rounds.
cd "$(dirname "$0")/.."
R=${R:-3}
cp paper_1909_04573_b200/libprnu.so /tmp/libA.so
for r in $(seq 1 $R); do
  for v in A B; do
    if [ $v = A ]; then cp /tmp/libA.so paper_1909_04573_b200/libprnu.so; else cp "$1" paper_1909_04573_b200/libprnu.so; fi
    timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-extras > gpurun_out/ablib_$v.json 2>/dev/null
    python tools/show_bench.py gpurun_out/ablib_$v.json 2>/dev/null | head -6 | sed "s/^/$v /"
  done
done
cp /tmp/libA.so paper_1909_04573_b200/libprnu.so
