#!/bin/bash
# Release build -> reference outputs; PRNU_DEBUG + PRNU_RACE_STRESS build -> the same
# workload must give bit-identical outputs (and no trapped bounds check); then the GPU
# test suite on the debug+stress build; finally the release build again.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python paper_1909_04573_b200/_build.py > /dev/null 2>&1 || { echo "release build failed"; exit 1; }
timeout 900 python tools/race_stress.py save gpurun_out/race_ref.pt || exit 1
PRNU_DEBUG=1 PRNU_NVCC_DEFS=PRNU_RACE_STRESS python paper_1909_04573_b200/_build.py > gpurun_out/stress_build.log 2>&1 || { echo "stress build failed"; tail gpurun_out/stress_build.log; exit 1; }
for rep in 1 2 3; do
  timeout 900 python tools/race_stress.py compare gpurun_out/race_ref.pt; echo "stress compare rc $?"
done
python -c "import paper_1909_04573_b200 as p; print('pytest against:', p.version())"
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_debug_stress.log 2>&1; echo "debug+stress pytest rc $?"; tail -2 gpurun_out/pytest_debug_stress.log
python paper_1909_04573_b200/_build.py > /dev/null 2>&1
