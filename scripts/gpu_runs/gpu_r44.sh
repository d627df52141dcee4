#!/bin/bash
# r44: GPU stress run of the dataset path vs the oracle (scripts/stress_dataset.py).
set -u
OUT=gpurun_out/r44
mkdir -p "$OUT"
timeout 2400 python scripts/stress_dataset.py --cases 6000 --seed 4242 > "$OUT/stress_dataset.jsonl" 2> "$OUT/stress.err"; echo "rc=$?" >> "$OUT/stress.err"
echo done > "$OUT/DONE"
