#!/bin/bash
# r15: full GPU suite, default bench, K5 persistent (software-pipelined) variants:
# same-box A/B + ncu.  Usage: gpurun -- 'bash scripts/gpu_runs/gpu_r15.sh'
set -u
TAG=${1:-r15}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 1500 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_gpu.log"
timeout 600 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
: > "$OUT/k5.jsonl"
for rep in 1 2; do
for m in lookback split persistent persistent3; do
  echo "{\"k5\": \"$m\", \"rep\": $rep}" >> "$OUT/k5.jsonl"
  RESHARD_K5=$m timeout 900 python bench.py --workload dataset-100m-dp2to4to8 --steps 10 --warmup 3 --no-cpu-baseline >> "$OUT/k5.jsonl" 2>> "$OUT/k5.err"
done
done
RESHARD_K5=persistent timeout 900 ncu --set full --clock-control none --import-source on -k regex:repartition_persistent -s 12 -c 1 \
  -o "$OUT/repart_persistent" python bench.py --workload dataset-100m-dp2to4to8 --steps 1 --warmup 3 --no-cpu-baseline \
  > "$OUT/ncu_dataset.log" 2>&1
echo done > "$OUT/DONE"
