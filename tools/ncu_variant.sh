#!/bin/bash
# ncu --set full of one level-1 launch of a variant tile kernel (regex $1, default k_var_syn2d) in
# tools/variant_profile.py 64 (first call: db4 symmetric; --launch-skip 3 = level 1), raw metrics grep'd.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
K=${1:-k_var_syn2d}; OUT=${2:-gpurun_out/var}
python tools/variant_profile.py 64 > /dev/null 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$K" --launch-skip ${SKIP:-3} -c 1 -f -o $OUT \
  python tools/variant_profile.py 64 > gpurun_out/ncu_var.log 2>&1
echo "ncu rc $?"
python tools/ncu_summary.py $OUT.ncu-rep
