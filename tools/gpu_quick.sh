#!/bin/bash
# quick GPU check: parity tests + short bench (no e2e / cpu baseline)
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/quick.json 2> gpurun_out/quick.err
echo "bench rc $?"; tail -3 gpurun_out/quick.err
python tools/show_bench.py gpurun_out/quick.json
