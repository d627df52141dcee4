#!/bin/bash
# r55: bulk_warp (32 lanes issue the per-row bulk copies) vs bulk_strided on the multi-row workloads.
set -u
OUT=gpurun_out/r55
mkdir -p "$OUT"
: > "$OUT/ab.jsonl"
for rep in 1 2; do
for k in bulk_strided bulk_warp; do
  for w in gpt2-small-tp2-to-pp2 gpt3-6.7b-tp4pp2-to-tp2pp2dp2; do
    echo "{\"kernel\": \"$k\", \"workload\": \"$w\", \"rep\": $rep}" >> "$OUT/ab.jsonl"
    RESHARD_COPY_KERNEL=$k timeout 900 python bench.py --workload $w --no-cpu-baseline --no-e2e >> "$OUT/ab.jsonl" 2>> "$OUT/err"
  done
done
done
echo done > "$OUT/DONE"
