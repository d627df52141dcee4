#!/bin/bash
# r50: memcheck over the executor suite with the device-side schedule expansion; 30k stress.
set -u
OUT=gpurun_out/r50
mkdir -p "$OUT"
S=/usr/local/cuda/bin/compute-sanitizer
timeout 2400 $S --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_executor.py -m gpu -x -q -k "not full_size and not config1" > "$OUT/memcheck_executor.log" 2>&1; echo "rc=$?" >> "$OUT/memcheck_executor.log"
timeout 2400 python scripts/stress_gpu.py --cases 30000 --seed 77 > "$OUT/stress_30k.jsonl" 2>&1
echo done > "$OUT/DONE"
