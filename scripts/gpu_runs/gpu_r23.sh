#!/bin/bash
# r23: GPT-3 6.7B (4,2,1)->(2,2,2) on one GPU in waves: bench, stage-shape sweep, ncu of one wave launch.
set -u
TAG=${1:-r23}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
W=gpt3-6.7b-tp4pp2-to-tp2pp2dp2
timeout 900 python bench.py --workload $W --steps 3 --warmup 3 --no-cpu-baseline > "$OUT/bench_67b.json" 2> "$OUT/bench_67b.err"
: > "$OUT/sweep.jsonl"
for cfg in "7 29" "6 32" "8 24" "4 48" "12 16"; do
  set -- $cfg
  echo "{\"stages\": $1, \"kib\": $2}" >> "$OUT/sweep.jsonl"
  RESHARD_BULK_STAGES=$1 RESHARD_BULK_STAGE_KIB=$2 timeout 600 python bench.py --workload $W --steps 3 --warmup 3 --no-cpu-baseline >> "$OUT/sweep.jsonl" 2>> "$OUT/sweep.err"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:copy_bulk -s 3 -c 1 \
  -o "$OUT/copy_67b" python bench.py --workload $W --steps 1 --warmup 1 --no-cpu-baseline > "$OUT/ncu_full.log" 2>&1
echo done > "$OUT/DONE"
