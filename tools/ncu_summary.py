"""Summarise an ncu --set full report (raw page CSV) per kernel: time, throughput, stalls, DRAM bytes."""
import csv
import subprocess
import sys

rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(txt.splitlines()))
hdr, units = r[0], r[1]
keys = ['gpu__time_duration.sum', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum',
        'smsp__inst_executed.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__occupancy_limit_shared_mem']
for row in r[2:]:
    vals = {h: row[i] for i, h in enumerate(hdr)}
    st = []
    for h, v in vals.items():
        if h.startswith('smsp__average_warps_issue_stalled_') and h.endswith('_per_issue_active.ratio'):
            try:
                st.append((h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''),
                           float(v.replace(',', ''))))
            except ValueError:
                pass
    st = sorted(st, key=lambda x: -x[1])[:7]
    print(row[hdr.index('ID')], vals['Kernel Name'][:60])
    print('   stalls:', [(h, round(v, 2)) for h, v in st])
    for k in keys:
        if k in vals:
            print('     ', k, vals[k], units[hdr.index(k)])
