#!/bin/bash
# r38: K5 with group / block sums (split2h, no tile-scan launch) — parity incl. full size + A/B.
set -u
OUT=gpurun_out/r38
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_dataset.py -m gpu -x -q > "$OUT/pytest_dataset.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_dataset.log"
RESHARD_K5=split2h timeout 900 python -m pytest tests/test_dataset.py -m gpu -x -q -k "full_size or host_buffer" > "$OUT/pytest_h.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_h.log"
for rep in 1 2; do
for m in split2 split2h; do
  echo "{\"k5\": \"$m\", \"rep\": $rep}" >> "$OUT/ab.jsonl"
  RESHARD_K5=$m timeout 300 python bench.py --workload dataset-100m-dp2to4to8 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> "$OUT/ab.jsonl" 2>> "$OUT/err"
done
done
echo done > "$OUT/DONE"
