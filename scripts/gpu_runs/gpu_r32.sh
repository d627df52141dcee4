#!/bin/bash
set -u
TAG=${1:-r32}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
for rep in 1 2; do
for m in split2 split2_6 split2_8; do
  echo "{\"k5\": \"$m\", \"rep\": $rep}" >> "$OUT/ab.jsonl"
  RESHARD_K5=$m timeout 300 python bench.py --workload dataset-100m-dp2to4to8 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> "$OUT/ab.jsonl" 2>> "$OUT/err"
done
done
echo done > "$OUT/DONE"
