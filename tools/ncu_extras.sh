#!/bin/bash
# ncu launch list of the NEXT-row kernels (f3 variants via tools/variant_profile.py)
cd "$(dirname "$0")/.."
O=gpurun_out/prof; mkdir -p $O
python tools/variant_profile.py > $O/variant_profile.txt 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/ncu_variants.csv python tools/variant_profile.py > /dev/null 2>&1; echo "ncu rc $?"
python tools/launch_summary.py $O/ncu_variants.csv > $O/ncu_variants_summary.txt
gzip -f $O/ncu_variants.csv
