#!/bin/bash
# A/B of the analysis kernels (PRNU_ANALYSIS=strip vs the default lifting kernel):
# residual parity tests first, then the short default bench for both.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc $?"; tail -15 gpurun_out/ab_pytest.log
for v in lift strip lift; do
  PRNU_ANALYSIS=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-extras > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  echo "== $v rc $?"; tail -2 gpurun_out/ab_$v.err; python tools/show_bench.py gpurun_out/ab_$v.json | head -9
done
