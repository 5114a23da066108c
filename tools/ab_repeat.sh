#!/bin/bash
# Interleaved repeated A/B of env settings: R rounds x each config, ms/step of each run.
# usage: R=3 bash tools/ab_repeat.sh "" "ENV=1" ...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
R=${R:-3}
for r in $(seq 1 $R); do
  i=0
  for envs in "$@"; do
    i=$((i+1))
    env $envs timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-extras --no-profile \
      > gpurun_out/abr_${i}_$r.json 2> /dev/null
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['ms_per_step'],3))" \
      gpurun_out/abr_${i}_$r.json "[$envs]"
  done
done
