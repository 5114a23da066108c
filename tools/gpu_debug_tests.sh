#!/bin/bash
# GPU test suite against a PRNU_DEBUG build (device-side PRNU_DCHECK bounds checks
# compiled in: a violated check traps the kernel), then the release build again.
cd "$(dirname "$0")/.."
PRNU_DEBUG=1 python paper_1909_04573_b200/_build.py --force > /dev/null 2>&1 || { echo "debug build failed"; exit 1; }
timeout 2000 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python paper_1909_04573_b200/_build.py --force > /dev/null 2>&1
