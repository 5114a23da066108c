#!/bin/bash
# Interleaved A/B/... of prebuilt libprnu.so files given as args, R rounds (default 3);
# each variant first runs the GPU parity file once.  The in-tree library is restored.
cd "$(dirname "$0")/.."
R=${R:-3}
cp paper_1909_04573_b200/libprnu.so /tmp/lib_intree.so
for v in "$@"; do
  cp "$v" paper_1909_04573_b200/libprnu.so
  echo "== parity $v: $(timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -1)"
done
for r in $(seq 1 $R); do
  for v in "$@"; do
    cp "$v" paper_1909_04573_b200/libprnu.so
    timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-extras > gpurun_out/abm.json 2>/dev/null
    python tools/show_bench.py gpurun_out/abm.json 2>/dev/null | head -5 | sed "s|^|$(basename $v) |"
  done
done
cp /tmp/lib_intree.so paper_1909_04573_b200/libprnu.so
