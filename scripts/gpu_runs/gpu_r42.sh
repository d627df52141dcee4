#!/bin/bash
# r42: compute-sanitizer over the executor suite (aux-stream concurrency, multi-GPU worlds,
# host-value slice / merge) and the multi-process dataset path.
set -u
OUT=gpurun_out/r42
mkdir -p "$OUT"
S=/usr/local/cuda/bin/compute-sanitizer
timeout 2400 $S --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_executor.py -m gpu -x -q -k "not full_size and not config1" > "$OUT/memcheck_executor.log" 2>&1; echo "rc=$?" >> "$OUT/memcheck_executor.log"
timeout 1800 $S --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_executor.py -m gpu -x -q -k "fig6 or single_process or host_value" > "$OUT/racecheck_executor.log" 2>&1; echo "rc=$?" >> "$OUT/racecheck_executor.log"
timeout 1800 $S --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_executor.py -m gpu -x -q -k "fig6 or single_process" > "$OUT/synccheck_executor.log" 2>&1; echo "rc=$?" >> "$OUT/synccheck_executor.log"
echo done > "$OUT/DONE"
