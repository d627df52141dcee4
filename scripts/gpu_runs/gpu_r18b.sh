#!/bin/bash
# r18b: K5 finalize variants (occupancy, 8 items per thread) — parity + same-box A/B.
set -u
TAG=${1:-r18b}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_dataset.py -m gpu -x -q > "$OUT/pytest_dataset.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_dataset.log"
: > "$OUT/ab.jsonl"
for rep in 1 2; do
for fin in def 8 6 it8; do
  echo "{\"fin\": \"$fin\", \"rep\": $rep}" >> "$OUT/ab.jsonl"
  RESHARD_K5_FIN=$fin timeout 300 python bench.py --workload dataset-100m-dp2to4to8 --steps 10 --warmup 3 --no-cpu-baseline >> "$OUT/ab.jsonl" 2>> "$OUT/ab.err"
done
done
echo done > "$OUT/DONE"
