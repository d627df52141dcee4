#!/bin/bash
# r73: long stress runs on the final tree (K8 rework included; new seeds)
set -u
OUT=gpurun_out/r73
mkdir -p "$OUT"
timeout 1800 python scripts/stress_k8.py --cases 3000 --seed 73 > "$OUT/stress_k8.jsonl" 2>&1
timeout 1500 python scripts/stress_dataset.py --cases 6000 --seed 7301 > "$OUT/stress_dataset_6k.jsonl" 2>&1
timeout 2400 python scripts/stress_gpu.py --cases 60000 --seed 7302 > "$OUT/stress_60k.jsonl" 2>&1
echo done > "$OUT/DONE"
