#!/bin/bash
# Default bench at the given depths (no extras / e2e / cpu baseline); prints the kernel table.
# usage: tools/depth_bench.sh 2 [1 ...]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for D in "$@"; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-extras --depths $D > gpurun_out/d$D.json 2> gpurun_out/d$D.err
  python - $D <<'PY'
import json, sys
d = json.loads(open("gpurun_out/d%s.json" % sys.argv[1]).read().strip().splitlines()[-1])
print("depth", sys.argv[1], "ms/step %.2f" % d["ms_per_step"], "value %.0f" % d["value"], d["unit"])
for k, v in d["kernels"].items():
    if v["ms_per_step"] > 0.1:
        print("   %-20s %7.3f ms %5.1f launches  %s GB/s" % (k, v["ms_per_step"], v["launches_per_step"], round(v.get("alg_GBps") or 0)))
PY
done
