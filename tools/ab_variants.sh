#!/bin/bash
# A/B compile-time variants on the GPU box: for each argument (a space-separated
# PRNU_NVCC_DEFS string, "" = default) rebuild the library and run a short bench.
cd "$(dirname "$0")/.."
for defs in "$@"; do
  echo "=== variant: '$defs'"
  PRNU_NVCC_DEFS="$defs" python paper_1909_04573_b200/_build.py --force > gpurun_out/ab_build.log 2>&1 || { echo build failed; tail -5 gpurun_out/ab_build.log; continue; }
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "bench rc $?"; tail -2 gpurun_out/ab.err
  python tools/show_bench.py gpurun_out/ab.json | head -8
done
python paper_1909_04573_b200/_build.py --force > /dev/null 2>&1
