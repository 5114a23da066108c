#!/bin/bash
# ncu throughput breakdowns (L1 / SM sub-units) of one launch of a kernel regex during
# tools/profile_extract.py, to see which L1 sub-unit l1tex__throughput's max comes from.
# usage: tools/ncu_breakdown.sh [kernel-regex] [out-name]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
K=${1:-k_analysis_lift}; OUT=${2:-gpurun_out/breakdown}
python tools/profile_extract.py 64 64 > /dev/null 2>&1 || { echo "plain run failed"; exit 1; }
timeout 600 ncu --clock-control none -k "regex:$K" --launch-skip ${SKIP:-0} -c 1 \
  --metrics breakdown:l1tex__throughput.avg.pct_of_peak_sustained_active,breakdown:sm__throughput.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts.sum,sm__cycles_elapsed.avg,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,launch__registers_per_thread,smsp__inst_executed_op_ldsm.sum,l1tex__data_bank_reads.sum,l1tex__data_bank_writes.sum,l1tex__lsuin_requests.sum,smsp__sass_inst_executed_op_shared_ld.sum,smsp__sass_inst_executed_op_shared_st.sum,smsp__sass_inst_executed_op_local_ld.sum,smsp__sass_inst_executed_op_local_st.sum \
  --csv python tools/profile_extract.py 64 64 > $OUT.csv 2> gpurun_out/ncu_breakdown.log
echo "ncu rc $?"; tail -2 gpurun_out/ncu_breakdown.log
python - "$OUT.csv" <<'EOF'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
for r in rows:
    if 'Metric Name' in r:
        hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        print(f"{d['Kernel Name'][:40]:40s} {d['Metric Name']:70s} {d['Metric Unit']:10s} {d['Metric Value']}")
EOF
