#!/bin/bash
set -u
TAG=${1:-r06}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 1200 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_gpu.log"
timeout 900 python bench.py --no-cpu-baseline > "$OUT/bench.json" 2> "$OUT/bench.err"
B="python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline"
: > "$OUT/sweep.jsonl"
for sv in "7 29" "8 24" "6 32" "8 26" "10 20" "12 16" "5 40"; do
  set -- $sv
  for w in gpt3-1.3b-dp-scaleout gpt2-small-tp2-to-pp2; do
    echo "{\"env\": \"stages=$1 kib=$2\", \"workload\": \"$w\"}" >> "$OUT/sweep.jsonl"
    RESHARD_BULK_STAGES=$1 RESHARD_BULK_STAGE_KIB=$2 timeout 300 $B --workload $w >> "$OUT/sweep.jsonl" 2>> "$OUT/sweep.err"
  done
done
timeout 1800 python bench.py --workload gpt3-6.7b-tp4pp2-to-tp2pp2dp2 --steps 3 --warmup 3 --no-cpu-baseline > "$OUT/bench_67b.json" 2> "$OUT/bench_67b.err"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:copy_bulk -s 3 -c 1 \
  -o "$OUT/copy_bulk" $B --steps 3 --warmup 3 > "$OUT/ncu_bulk.log" 2>&1
echo done > "$OUT/DONE"
