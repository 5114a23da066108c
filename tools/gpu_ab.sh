#!/bin/bash
# parity tests (fast subset unless FULL=1) + bench A/B of env settings given as args ("" = default)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
if [ -n "$FULL" ]; then timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5;
else timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -5; fi
i=0
for envs in "$@"; do
  i=$((i+1))
  env $envs timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-extras > gpurun_out/ab_$i.json 2> gpurun_out/ab_$i.err
  echo "== [$envs] rc $?"; tail -2 gpurun_out/ab_$i.err
  python tools/show_bench.py gpurun_out/ab_$i.json | head -8
done
