#!/bin/bash
# ncu --set full of the first N launches of a kernel regex during tools/profile_extract.py
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
K=${1:-k_analysis_strip}; C=${2:-4}; OUT=${3:-gpurun_out/strip}
python tools/profile_extract.py 64 64 > /dev/null 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$K" --launch-skip ${SKIP:-0} -c $C -f -o $OUT python tools/profile_extract.py 64 64 > gpurun_out/ncu_strip.log 2>&1
echo "ncu rc $?"; tail -3 gpurun_out/ncu_strip.log
python tools/ncu_summary.py $OUT.ncu-rep
