#!/bin/bash
# Round evidence in one GPU call: build + smoke, the whole GPU suite, profile collection.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/prof
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -12 gpurun_out/pytest_gpu.log
bash tools/collect_profiles.sh
