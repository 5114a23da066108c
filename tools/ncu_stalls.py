"""Stall-reason shares and a few headline metrics of the first kernel in an ncu report:
   python tools/ncu_stalls.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
d = dict(zip(rows[0], rows[2]))
pre = "smsp__pcsamp_warps_issue_stalled_"
st = {k[len(pre):]: float(v.replace(",", "")) for k, v in d.items()
      if k.startswith(pre) and not k.endswith("not_issued") and v.replace(",", "").replace(".", "").isdigit()}
tot = sum(st.values()) or 1.0
print("stalls:", ", ".join(f"{k} {v / tot:.2f}" for k, v in sorted(st.items(), key=lambda x: -x[1]) if v / tot > 0.02))
for k in ("gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "dram__bytes_read.sum", "dram__bytes_write.sum"):
    print(f"  {k} {d.get(k)}")
