#!/bin/bash
set -u
OUT=gpurun_out/r47b
mkdir -p "$OUT"
RESHARD_HOST_TRACE=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 > "$OUT/bench.json" 2> "$OUT/trace.err"
echo done > "$OUT/DONE"
