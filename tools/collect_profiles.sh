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
python tools/ncu_opmix.py $O/full.ncu-rep "k_analysis_lift" 33466176 > $O/ncu_opmix_analysis_l1.txt
python tools/ncu_lines.py $O/full.ncu-rep "k_analysis_lift" 40 > $O/ncu_lines_analysis_l1.txt
echo done
# PCE (camera-ID cached call, 64 pairs 720x1280): launch list + full capture of the column kernel
python tools/pce_batch_once.py > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum \
  --clock-control none --csv python tools/pce_batch_once.py > $O/pce_launches.csv 2> $O/pce_launches.err; echo "pce list rc $?"
python tools/ncu_agg.py $O/pce_launches.csv > $O/ncu_pce_launches.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pce_cols -s 1 -c 1 -f -o $O/pce_cols \
  python tools/pce_batch_once.py > $O/pce_full_run.log 2>&1; echo "pce full rc $?"
python tools/ncu_kstats.py $O/pce_cols.ncu-rep > $O/ncu_pce_cols_summary.txt
python tools/ncu_stall_lines.py $O/pce_cols.ncu-rep k_pce_cols 20 >> $O/ncu_pce_cols_summary.txt
echo pce done
