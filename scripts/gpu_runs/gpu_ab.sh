#!/bin/bash
# Same-box A/B of copy-kernel variants.  Usage: gpurun -- 'bash scripts/gpu_ab.sh <tag>'
set -u
TAG=${1:-ab}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
B="python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline"
: > "$OUT/ab.jsonl"
for rep in 1 2; do
for k in bulk bulk_strided; do
  for sv in "7 29" "8 24" "6 32"; do
    set -- $sv
    for w in gpt3-1.3b-dp-scaleout gpt2-small-tp2-to-pp2; do
      echo "{\"env\": \"$k stages=$1 kib=$2 rep=$rep\", \"workload\": \"$w\"}" >> "$OUT/ab.jsonl"
      RESHARD_COPY_KERNEL=$k RESHARD_BULK_STAGES=$1 RESHARD_BULK_STAGE_KIB=$2 timeout 300 $B --workload $w >> "$OUT/ab.jsonl" 2>> "$OUT/ab.err"
    done
  done
done
done
for k in bulk bulk_strided ldg; do
  echo "{\"env\": \"$k 6.7b\", \"workload\": \"67b\"}" >> "$OUT/ab.jsonl"
  RESHARD_COPY_KERNEL=$k timeout 900 python bench.py --workload gpt3-6.7b-tp4pp2-to-tp2pp2dp2 --steps 3 --warmup 3 --no-cpu-baseline >> "$OUT/ab.jsonl" 2>> "$OUT/ab.err"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:copy_bulk -s 3 -c 1 \
  -o "$OUT/copy_bulk" $B --steps 3 --warmup 3 > "$OUT/ncu_bulk.log" 2>&1
RESHARD_COPY_KERNEL=bulk_strided timeout 900 ncu --set full --clock-control none --import-source on -k regex:copy_bulk -s 3 -c 1 \
  -o "$OUT/copy_bulk_strided" $B --steps 3 --warmup 3 > "$OUT/ncu_bulk_strided.log" 2>&1
echo done > "$OUT/DONE"
