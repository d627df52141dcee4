#!/bin/bash
set -u
OUT=gpurun_out/r40
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_cpp_api.py tests/test_gpu_executor.py -m gpu -x -q > "$OUT/pytest.log" 2>&1; echo "rc=$?" >> "$OUT/pytest.log"
echo done > "$OUT/DONE"
