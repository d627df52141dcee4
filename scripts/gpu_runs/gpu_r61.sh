#!/bin/bash
set -u
OUT=gpurun_out/r61
mkdir -p "$OUT"
df -h /dev/shm > "$OUT/shm.txt" 2>&1; free -g >> "$OUT/shm.txt" 2>&1
timeout 900 python scripts/probe_checkpoint.py > "$OUT/checkpoint.jsonl" 2>&1
echo done > "$OUT/DONE"
