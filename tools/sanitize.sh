#!/bin/bash
# One compute-sanitizer tool per call (B200_PROFILING.md): plain run first, then the tool.
# usage: tools/sanitize.sh memcheck|racecheck|synccheck|initcheck [--quick]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TOOL=$1; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python tools/sanitize_run.py "$@" > gpurun_out/sanitize_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/sanitize_plain.log; exit 1; }
EXTRA=""
[ "$TOOL" = "racecheck" ] && EXTRA="--racecheck-report hazard"
[ "$TOOL" = "memcheck" ] && EXTRA="--leak-check no"
timeout 2400 compute-sanitizer --tool $TOOL $EXTRA --print-limit 50 python tools/sanitize_run.py "$@" > gpurun_out/sanitize_$TOOL.log 2>&1
echo "sanitizer rc $?"
tail -4 gpurun_out/sanitize_$TOOL.log
