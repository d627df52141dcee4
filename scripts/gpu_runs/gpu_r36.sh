#!/bin/bash
set -u
OUT=gpurun_out/r36
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_gpu_executor.py -m gpu -x -q > "$OUT/pytest_executor.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_executor.log"
echo done > "$OUT/DONE"
