#!/bin/bash
# r58: bulk_strided CTA count / stage shape sweep on the default workload (same box).
set -u
OUT=gpurun_out/r58b
mkdir -p "$OUT"
: > "$OUT/sweep.jsonl"
for rep in 1 2; do
for cfg in "1 7 29" "1 7 28" "1 7 30" "1 7 31"; do
  set -- $cfg
  echo "{\"ctas\": $1, \"stages\": $2, \"kib\": $3, \"rep\": $rep}" >> "$OUT/sweep.jsonl"
  RESHARD_CTAS_PER_SM=$1 RESHARD_BULK_STAGES=$2 RESHARD_BULK_STAGE_KIB=$3 timeout 300 python bench.py --no-cpu-baseline --no-e2e >> "$OUT/sweep.jsonl" 2>> "$OUT/err"
done
done
echo done > "$OUT/DONE"
