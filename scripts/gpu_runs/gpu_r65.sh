#!/bin/bash
set -u
OUT=gpurun_out/r65
mkdir -p "$OUT"
for i in 1 2; do RESHARD_HOST_TRACE=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 > "$OUT/bench_$i.json" 2> "$OUT/trace_$i.err"; done
echo done > "$OUT/DONE"
