#!/bin/bash
# Short default bench (no extras) + the per-kernel table; for A/B of kernel configurations.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-extras > gpurun_out/quick.json 2> gpurun_out/quick.err
echo "bench rc $?"; tail -1 gpurun_out/quick.err
python tools/show_bench.py gpurun_out/quick.json 2>/dev/null | head -${ROWS:-12}
