import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
ks = d.pop("kernels", None) or {}
print(f"value {d['value']:.1f} {d['unit']}  ms/step {d['ms_per_step']:.2f}  clocks {d.get('clocks')}")
if d.get("roofline"):
    r = d["roofline"]
    print(f"roofline {r['kernel']} {r['bound']} {r['achieved']:.1f} {r['unit']} frac {r['frac']:.3f} share {r['share_of_kernel_time']:.3f}"
          + (f" | alu {r['alu_view']['achieved']:.1f} T lane-op/s frac {r['alu_view']['frac']:.3f}" if r.get('alu_view') else ""))
for k, v in sorted(ks.items(), key=lambda x: -x[1]["ms_per_step"]):
    print(f"{k:20s} {v['ms_per_step']:8.3f} ms {v['launches_per_step']:7.1f} launches share {v['share']:.3f} "
          f"{v.get('alg_GBps', 0):8.1f} GB/s")
for key in ("e2e", "cpu_baseline", "ncc_vs_true_K"):
    if d.get(key):
        print(key, d[key])
