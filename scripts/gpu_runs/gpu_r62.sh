#!/bin/bash
set -u
OUT=gpurun_out/r62
mkdir -p "$OUT"
timeout 600 python bench.py --no-cpu-baseline > "$OUT/bench.json" 2> "$OUT/bench.err"
timeout 900 python bench.py --workload gpt3-6.7b-tp4pp2-to-tp2pp2dp2 --no-cpu-baseline > "$OUT/bench_67b.json" 2>> "$OUT/bench.err"
echo done > "$OUT/DONE"
