#!/bin/bash
set -u
OUT=gpurun_out/r60
mkdir -p "$OUT"
timeout 1800 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python __graft_entry__.py --smoke > "$OUT/smoke.log" 2>&1; echo "rc=$?" >> "$OUT/smoke.log"
echo done > "$OUT/DONE"
