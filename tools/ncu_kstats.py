"""Per-kernel headline metrics and stall shares of every kernel in an ncu report:
   python tools/ncu_kstats.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
pre = "smsp__pcsamp_warps_issue_stalled_"
for v in rows[2:]:
    d = dict(zip(h, v))
    st = {k[len(pre):]: float(x.replace(",", "")) for k, x in d.items()
          if k.startswith(pre) and not k.endswith("not_issued") and x.replace(",", "").replace(".", "").isdigit()}
    tot = sum(st.values()) or 1.0
    print(d["Kernel Name"][:70], "| us", d["gpu__time_duration.sum"], "| inst", d["smsp__inst_executed.sum"],
          "| issue%", d["smsp__issue_active.avg.pct_of_peak_sustained_active"], "| dram MB",
          d["dram__bytes_read.sum"], d["dram__bytes_write.sum"], "| warps%",
          d["sm__warps_active.avg.pct_of_peak_sustained_active"], "| smem wf",
          d.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"))
    print("    stalls:", ", ".join(f"{k} {x / tot:.2f}" for k, x in sorted(st.items(), key=lambda z: -z[1])
                                   if x / tot > 0.03))
