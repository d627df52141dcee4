#!/bin/bash
set -u
OUT=gpurun_out/r33c
mkdir -p "$OUT"
timeout 900 python bench.py --workload dataset-100m-dp2to4to8 --steps 10 --warmup 3 > "$OUT/bench_dataset.json" 2> "$OUT/err"
timeout 600 python -m pytest tests/test_gpu_multiprocess.py -m gpu -x -q > "$OUT/pytest_mp.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_mp.log"
echo done > "$OUT/DONE"
