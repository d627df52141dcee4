#!/bin/bash
# r67b: windowed K8, smaller windows
set -u
OUT=gpurun_out/r67b
mkdir -p "$OUT"
timeout 900 python scripts/probe_k8.py --fracs 80,160,320,640,1280 > "$OUT/probe_k8.jsonl" 2> "$OUT/probe_k8.err"
timeout 600 python scripts/probe_k8.py --n 3000000 --fracs 20,40,80,160 > "$OUT/probe_k8_3m.jsonl" 2>> "$OUT/probe_k8.err"
echo done > "$OUT/DONE"
