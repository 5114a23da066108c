#!/bin/bash
# GPU check: smoke, the GPU test suite (optionally -k filter), short default bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/smoke.log
timeout ${PYTEST_TIMEOUT:-1500} python -m pytest tests -m gpu -x -q -s ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
grep -E "C2 d=|passed|failed|Error|error" gpurun_out/pytest_gpu.log | tail -12
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-extras > gpurun_out/quick.json 2> gpurun_out/quick.err
echo "bench rc $?"; tail -2 gpurun_out/quick.err
python tools/show_bench.py gpurun_out/quick.json 2>/dev/null | head -16
