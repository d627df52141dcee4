#!/bin/bash
set -u
OUT=gpurun_out/r46
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_gpu_multiprocess.py -m gpu -x -q > "$OUT/pytest_mp.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_mp.log"
timeout 600 python bench.py --no-cpu-baseline > "$OUT/bench.json" 2> "$OUT/bench.err"
timeout 900 python bench.py --workload gpt3-6.7b-tp4pp2-to-tp2pp2dp2 --no-cpu-baseline > "$OUT/bench_67b.json" 2>> "$OUT/bench.err"
echo done > "$OUT/DONE"
