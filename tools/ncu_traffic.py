"""DRAM bytes of the first launch of a kernel in an ncu --set full report -> traffic.json
usage: ncu_traffic.py report.ncu-rep kernel_regex bench_kernel_name frames_per_launch H W source_note"""
import csv, json, re, subprocess, sys
rep, kre, bname, fpl, H, W, note = sys.argv[1:8]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(txt.splitlines()))
hdr, units = r[0], r[1]
for row in r[2:]:
    v = dict(zip(hdr, row))
    if re.search(kre, v["Kernel Name"]):
        def mb(k):
            x = float(v[k].replace(",", ""))
            u = units[hdr.index(k)]
            return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
        out = {"source": note, "kernel": bname, "ncu_kernel": v["Kernel Name"][:80], "frames_per_launch": int(fpl),
               "H": int(H), "W": int(W), "dram_bytes_read": mb("dram__bytes_read.sum"),
               "dram_bytes_write": mb("dram__bytes_write.sum"),
               "gpu_time_us_under_ncu": float(v["gpu__time_duration.sum"].replace(",", "")) }
        print(json.dumps(out, indent=1))
        break
