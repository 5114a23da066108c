#!/bin/bash
# Round profile evidence (one GPU): default bench line, ncu launch list of the bench,
# ncu --set full of one depth-1 wave (batch 64) of the extraction kernels.
cd "$(dirname "$0")/.."
O=gpurun_out/prof; mkdir -p $O
timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench.err; echo "bench rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ncu_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-profile --no-extras > $O/ncu_launch_run.log 2>&1; echo "ncu list rc $?"
python tools/launch_summary.py $O/ncu_launches.csv > $O/ncu_launches_summary.txt
gzip -f $O/ncu_launches.csv
python tools/profile_extract.py 64 64 > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k "regex:k_analysis_lift|k_synth_acc2|k_sda_sum" -c 9 -f -o $O/full \
  python tools/profile_extract.py 64 64 > $O/ncu_full_run.log 2>&1; echo "ncu full rc $?"
python tools/ncu_summary.py $O/full.ncu-rep > $O/ncu_full_summary.txt
python tools/ncu_traffic.py $O/full.ncu-rep "k_analysis_lift<unsigned char" analysis_l1_u8 64 1080 1920 \
  "profiles/r02/full.ncu-rep: k_analysis_lift<u8> (analysis_l1_u8), FHD, 64 frames per launch" > $O/traffic.json
python tools/ncu_opmix.py $O/full.ncu-rep "k_analysis_lift<unsigned char" 33466176 > $O/ncu_opmix_analysis_l1.txt
python tools/ncu_lines.py $O/full.ncu-rep "k_analysis_lift<unsigned char" 40 > $O/ncu_lines_analysis_l1.txt
echo done
