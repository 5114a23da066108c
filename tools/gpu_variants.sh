#!/bin/bash
# Build-time variants: for each arg (space-separated -D defs, "" = default), rebuild and bench quickly
# (VTEST=1: also run the parity tests on each variant).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
i=0
for defs in "$@"; do
  i=$((i+1))
  PRNU_NVCC_DEFS="$defs" python paper_1909_04573_b200/_build.py --force > gpurun_out/var_build_$i.log 2>&1 || { echo "build $i failed"; tail -5 gpurun_out/var_build_$i.log; continue; }
  [ -n "$VTEST" ] && { timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2; }
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-extras > gpurun_out/var_$i.json 2> gpurun_out/var_$i.err
  echo "== [$defs] rc $?"; tail -2 gpurun_out/var_$i.err
  python tools/show_bench.py gpurun_out/var_$i.json 2>/dev/null | head -8
done
python paper_1909_04573_b200/_build.py --force > /dev/null 2>&1
