#!/bin/bash
set -u
TAG=${1:-r29}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
RESHARD_HOST_TRACE=1 timeout 300 python bench.py --workload gpt2-small-tp2-to-pp2 --no-cpu-baseline --e2e-steps 1 > "$OUT/gpt2.json" 2> "$OUT/gpt2_trace.err"
RESHARD_HOST_TRACE=1 timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 > "$OUT/default.json" 2> "$OUT/default_trace.err"
echo done > "$OUT/DONE"
