#!/bin/bash
# r16e: K5 lookback / pipe / pipe_nolb (diagnostic) and gather-only vs gather+write floor probes.
set -u
TAG=${1:-r16e}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
: > "$OUT/k5.jsonl"
for m in lookback pipe pipe_nolb; do
for pr in read write; do
  echo "{\"k5\": \"$m\", \"probe\": \"$pr\"}" >> "$OUT/k5.jsonl"
  RESHARD_K5=$m RESHARD_PROBE=$pr timeout 300 python bench.py --workload dataset-100m-dp2to4to8 --steps 5 --warmup 3 --no-cpu-baseline >> "$OUT/k5.jsonl" 2>> "$OUT/k5.err"
done
done
RESHARD_K5=pipe RESHARD_PROBE=write timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"probe|repartition" \
  --csv --log-file "$OUT/launches.csv" python bench.py --workload dataset-100m-dp2to4to8 --steps 3 --warmup 3 --no-cpu-baseline > "$OUT/ncu.log" 2>&1
echo done > "$OUT/DONE"
