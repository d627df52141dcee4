#!/bin/bash
set -u
TAG=${1:-r29b}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
for c in 8 16 24 32 64; do
  echo "{\"chunks\": $c}" >> "$OUT/gpt2.jsonl"
  RESHARD_HOST_CHUNKS=$c timeout 300 python bench.py --workload gpt2-small-tp2-to-pp2 --no-cpu-baseline --e2e-steps 5 >> "$OUT/gpt2.jsonl" 2>> "$OUT/err"
done
echo done > "$OUT/DONE"
