#!/bin/bash
# Round-1 check #4: multi-process IPC on one GPU, 6.7B waves, dataset K5 v3, finer bulk sweep.
set -u
TAG=${1:-r04}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 1200 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_gpu.log"
timeout 900 python bench.py --workload dataset-100m-dp2to4to8 --steps 10 --warmup 3 > "$OUT/bench_dataset.json" 2>&1
B="python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline"
: > "$OUT/sweep.jsonl"
for sv in "7 28" "7 30" "7 32" "6 32" "8 27" "5 40" "4 56" "7 29" "14 14"; do
  set -- $sv
  for w in gpt3-1.3b-dp-scaleout gpt2-small-tp2-to-pp2; do
    echo "{\"env\": \"stages=$1 kib=$2\", \"workload\": \"$w\"}" >> "$OUT/sweep.jsonl"
    RESHARD_BULK_STAGES=$1 RESHARD_BULK_STAGE_KIB=$2 timeout 300 $B --workload $w >> "$OUT/sweep.jsonl" 2>> "$OUT/sweep.err"
  done
done
echo "{\"env\": \"ctas=2 stages=7 kib=14\"}" >> "$OUT/sweep.jsonl"
RESHARD_CTAS_PER_SM=2 RESHARD_BULK_STAGES=7 RESHARD_BULK_STAGE_KIB=14 timeout 300 $B >> "$OUT/sweep.jsonl" 2>> "$OUT/sweep.err"
timeout 1800 python bench.py --workload gpt3-6.7b-tp4pp2-to-tp2pp2dp2 --steps 3 --warmup 3 --no-cpu-baseline > "$OUT/bench_67b.json" 2> "$OUT/bench_67b.err"
timeout 1800 python bench.py --workload gpt3-6.7b-recovery --steps 3 --warmup 3 --no-cpu-baseline > "$OUT/bench_67b_recovery.json" 2> "$OUT/bench_67b_recovery.err"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:repartition -s 4 -c 1 \
  -o "$OUT/repartition" python bench.py --workload dataset-100m-dp2to4to8 --steps 1 --warmup 3 --no-cpu-baseline \
  > "$OUT/ncu_dataset.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:shuffle -s 10 -c 3 \
  -o "$OUT/shuffle" python bench.py --workload dataset-100m-dp2to4to8 --steps 1 --warmup 3 --no-cpu-baseline \
  > "$OUT/ncu_shuffle.log" 2>&1
echo done > "$OUT/DONE"
