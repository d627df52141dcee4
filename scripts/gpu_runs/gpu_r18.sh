#!/bin/bash
# r18: padded 32-byte index layout — dataset GPU tests, same-box A/B packed vs padded, launch list.
set -u
TAG=${1:-r18}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_dataset.py -m gpu -x -q > "$OUT/pytest_dataset.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_dataset.log"
: > "$OUT/ab.jsonl"
for rep in 1 2; do
for lay in packed padded; do
  echo "{\"index\": \"$lay\", \"rep\": $rep}" >> "$OUT/ab.jsonl"
  RESHARD_INDEX=$lay timeout 300 python bench.py --workload dataset-100m-dp2to4to8 --steps 10 --warmup 3 --no-cpu-baseline >> "$OUT/ab.jsonl" 2>> "$OUT/ab.err"
done
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"repart|probe|pad" \
  --csv --log-file "$OUT/launches_dataset.csv" python bench.py --workload dataset-100m-dp2to4to8 --steps 3 --warmup 3 --no-cpu-baseline > "$OUT/ncu_launches.log" 2>&1
echo done > "$OUT/DONE"
