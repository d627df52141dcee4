#!/bin/bash
# r63: long stress runs on the final code path (new seeds).
set -u
OUT=gpurun_out/r63
mkdir -p "$OUT"
timeout 2400 python scripts/stress_gpu.py --cases 150000 --seed 1001 > "$OUT/stress_150k.jsonl" 2>&1
timeout 1500 python scripts/stress_dataset.py --cases 12000 --seed 2002 > "$OUT/stress_dataset_12k.jsonl" 2>&1
echo done > "$OUT/DONE"
