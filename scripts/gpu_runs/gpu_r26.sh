#!/bin/bash
# r26: bulk + LDG kernels on two streams (concurrent local relayout and peer pushes) — GPU suite.
set -u
TAG=${1:-r26}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 1800 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_gpu.log"
timeout 600 python bench.py --no-cpu-baseline > "$OUT/bench.json" 2> "$OUT/bench.err"
echo done > "$OUT/DONE"
