#!/bin/bash
# Bench with the next-row extras (configs 3-5, f1-f4) but no e2e / cpu baseline; prints the C5 sweep and C4.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/extras.json 2> gpurun_out/extras.err
echo "bench rc $?"; tail -1 gpurun_out/extras.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/extras.json").read().strip().splitlines()[-1])
print("step", round(d["ms_per_step"], 2), "ms", round(d["value"]), d["unit"])
nr = d.get("next_rows", {})
for k, v in nr.get("c5_depth_sweep", {}).items():
    print("c5 d=%s" % k, {kk: (round(vv, 3) if isinstance(vv, float) else vv) for kk, vv in v.items()})
print("c4", nr.get("c4_camera_id"))
for k, v in nr.get("f3_variants", {}).items():
    print("f3", k, v)
PY
