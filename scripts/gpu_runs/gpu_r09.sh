#!/bin/bash
set -u
TAG=${1:-r09}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 600 python __graft_entry__.py --smoke > "$OUT/smoke.log" 2>&1; echo "rc=$?" >> "$OUT/smoke.log"
timeout 1500 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_gpu.log"
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
B="python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline"
: > "$OUT/ab.jsonl"
for k in bulk_strided bulk; do
  for sv in "6 32" "7 29" "5 40" "4 48"; do
    set -- $sv
    for w in gpt3-1.3b-dp-scaleout gpt2-small-tp2-to-pp2; do
      echo "{\"env\": \"$k stages=$1 kib=$2\", \"workload\": \"$w\"}" >> "$OUT/ab.jsonl"
      RESHARD_COPY_KERNEL=$k RESHARD_BULK_STAGES=$1 RESHARD_BULK_STAGE_KIB=$2 timeout 300 $B --workload $w >> "$OUT/ab.jsonl" 2>> "$OUT/ab.err"
    done
  done
done
timeout 1800 python bench.py --workload gpt3-6.7b-tp4pp2-to-tp2pp2dp2 --steps 3 --warmup 3 --no-cpu-baseline > "$OUT/bench_67b.json" 2> "$OUT/bench_67b.err"
timeout 1800 python bench.py --workload gpt3-6.7b-recovery --steps 3 --warmup 3 --no-cpu-baseline > "$OUT/bench_67b_recovery.json" 2> "$OUT/bench_67b_recovery.err"
timeout 900 python bench.py --workload gpt2-small-tp2-to-pp2 --steps 20 --warmup 5 > "$OUT/bench_gpt2.json" 2>&1
timeout 900 python bench.py --workload dataset-100m-dp2to4to8 --steps 10 --warmup 3 > "$OUT/bench_dataset.json" 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
  $B --steps 3 --warmup 3 > "$OUT/ncu_launch.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:copy_bulk -s 3 -c 1 \
  -o "$OUT/copy_bulk_strided" $B --steps 3 --warmup 3 > "$OUT/ncu_bulk.log" 2>&1
echo done > "$OUT/DONE"
