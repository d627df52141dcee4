#!/bin/bash
set -u
TAG=${1:-r21b}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_dataset.py -m gpu -x -q > "$OUT/pytest_dataset.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_dataset.log"
for rep in 1 2; do
timeout 300 python bench.py --workload dataset-100m-dp2to4to8 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> "$OUT/bench.jsonl" 2>> "$OUT/bench.err"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"repart|probe" \
  --csv --log-file "$OUT/launches_dataset.csv" python bench.py --workload dataset-100m-dp2to4to8 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > "$OUT/ncu_launches.log" 2>&1
echo done > "$OUT/DONE"
