#!/bin/bash
# r39: the reference's value-level Tensor / slice / merge through the GPU (C++ and C ABI) + GPU suite.
set -u
OUT=gpurun_out/r39
mkdir -p "$OUT"
timeout 1800 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_gpu.log"
echo done > "$OUT/DONE"
