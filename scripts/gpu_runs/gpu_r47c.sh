#!/bin/bash
set -u
OUT=gpurun_out/r47c
mkdir -p "$OUT"
for t in 1 16; do
  RESHARD_HOST_THREADS=$t RESHARD_HOST_TRACE=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 > "$OUT/bench_$t.json" 2> "$OUT/trace_$t.err"
  RESHARD_HOST_THREADS=$t timeout 900 python bench.py --workload gpt3-6.7b-tp4pp2-to-tp2pp2dp2 --no-cpu-baseline --steps 3 > "$OUT/bench67_$t.json" 2>> "$OUT/trace_$t.err"
done
echo done > "$OUT/DONE"
