#!/bin/bash
# r16: K5 pipelined (cp.async, double-buffered) variant: parity + same-box A/B + ncu.
set -u
TAG=${1:-r16}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 600 python -m pytest tests/test_dataset.py -m gpu -x -q -k "pipe or lookback" > "$OUT/pytest_dataset.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_dataset.log"
: > "$OUT/k5.jsonl"
for rep in 1 2; do
for m in lookback pipe; do
  echo "{\"k5\": \"$m\", \"rep\": $rep}" >> "$OUT/k5.jsonl"
  RESHARD_K5=$m timeout 300 python bench.py --workload dataset-100m-dp2to4to8 --steps 10 --warmup 3 --no-cpu-baseline >> "$OUT/k5.jsonl" 2>> "$OUT/k5.err"
done
done
RESHARD_K5=pipe timeout 600 ncu --set full --clock-control none --import-source on -k regex:repartition_pipe -s 12 -c 1 \
  -o "$OUT/repart_pipe" python bench.py --workload dataset-100m-dp2to4to8 --steps 1 --warmup 3 --no-cpu-baseline \
  > "$OUT/ncu_dataset.log" 2>&1
echo done > "$OUT/DONE"
