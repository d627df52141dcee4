#!/bin/bash
set -u
TAG=${1:-r16c}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
: > "$OUT/k5.jsonl"
for m in lookback pipe pipe_nolb split; do
  echo "{\"k5\": \"$m\", \"rep\": 1}" >> "$OUT/k5.jsonl"
  RESHARD_K5=$m timeout 300 python bench.py --workload dataset-100m-dp2to4to8 --steps 10 --warmup 3 --no-cpu-baseline >> "$OUT/k5.jsonl" 2>> "$OUT/k5.err"
done
RESHARD_K5=split timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:repart_ \
  --csv --log-file "$OUT/split_launches.csv" python bench.py --workload dataset-100m-dp2to4to8 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
echo done > "$OUT/DONE"
