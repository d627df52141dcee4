#!/bin/bash
# r16f: K5 split2 (register-light gather pass) parity + A/B against the single-pass default.
set -u
TAG=${1:-r16f}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 600 python -m pytest tests/test_dataset.py -m gpu -x -q -k "split2 or lookback" > "$OUT/pytest_dataset.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_dataset.log"
: > "$OUT/k5.jsonl"
for rep in 1 2; do
for m in lookback split2 split2_6 split2_5; do
  echo "{\"k5\": \"$m\", \"rep\": $rep}" >> "$OUT/k5.jsonl"
  RESHARD_K5=$m RESHARD_PROBE=write timeout 300 python bench.py --workload dataset-100m-dp2to4to8 --steps 10 --warmup 3 --no-cpu-baseline >> "$OUT/k5.jsonl" 2>> "$OUT/k5.err"
done
done
RESHARD_K5=split2_5 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"repart" \
  --csv --log-file "$OUT/launches.csv" python bench.py --workload dataset-100m-dp2to4to8 --steps 3 --warmup 3 --no-cpu-baseline > "$OUT/ncu.log" 2>&1
echo done > "$OUT/DONE"
