#!/bin/bash
# Round-1 check #3: tests, default (bulk) bench with e2e, bulk stage sweep, gpt2/dataset, ncu.
set -u
TAG=${1:-r03}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 600 python __graft_entry__.py --smoke > "$OUT/smoke.log" 2>&1; echo "rc=$?" >> "$OUT/smoke.log"
timeout 1200 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_gpu.log"
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
B="python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline"
: > "$OUT/sweep.jsonl"
for sv in "8 24" "9 24" "10 20" "7 28" "8 26" "11 18" "6 36"; do
  set -- $sv
  echo "{\"env\": \"stages=$1 kib=$2\"}" >> "$OUT/sweep.jsonl"
  RESHARD_BULK_STAGES=$1 RESHARD_BULK_STAGE_KIB=$2 timeout 300 $B >> "$OUT/sweep.jsonl" 2>> "$OUT/sweep.err"
done
for w in gpt2-small-tp2-to-pp2; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 > "$OUT/bench_$w.json" 2>&1
  RESHARD_COPY_KERNEL=ldg timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > "$OUT/bench_${w}_ldg.json" 2>&1
done
timeout 900 python bench.py --workload dataset-100m-dp2to4to8 --steps 10 --warmup 3 > "$OUT/bench_dataset.json" 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
  $B --steps 3 --warmup 3 > "$OUT/ncu_launch.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:copy_bulk -s 3 -c 1 \
  -o "$OUT/copy_bulk" $B --steps 3 --warmup 3 > "$OUT/ncu_bulk.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:repartition -s 4 -c 1 \
  -o "$OUT/repartition" python bench.py --workload dataset-100m-dp2to4to8 --steps 1 --warmup 3 --no-cpu-baseline \
  > "$OUT/ncu_dataset.log" 2>&1
echo done > "$OUT/DONE"
