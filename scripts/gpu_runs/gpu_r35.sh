#!/bin/bash
set -u
OUT=gpurun_out/r35
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_gpu_executor.py -m gpu -x -q -k "single_process_multi_gpu" > "$OUT/pytest.log" 2>&1; echo "rc=$?" >> "$OUT/pytest.log"
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_executor.py -m gpu -x -q -k "single_process_multi_gpu and 4" > "$OUT/memcheck.log" 2>&1; echo "rc=$?" >> "$OUT/memcheck.log"
echo done > "$OUT/DONE"
