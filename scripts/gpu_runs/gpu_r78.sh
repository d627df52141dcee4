#!/bin/bash
# r78: K8 geometric window (lo/20 clamped to [64 Ki, N/20]) vs the fixed N/160 window
set -u
OUT=gpurun_out/r78
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_dataset.py -m gpu -x -q > "$OUT/pytest_dataset.log" 2>&1
timeout 900 python scripts/stress_k8.py --cases 1500 --seed 78 > "$OUT/stress_k8.jsonl" 2>&1
timeout 600 python scripts/probe_k8.py --fracs 0,160,0,160 > "$OUT/probe_k8.jsonl" 2> "$OUT/probe_k8.err"
RESHARD_K8_DIV=40 timeout 600 python scripts/probe_k8.py --fracs 0 > "$OUT/probe_k8_div40.jsonl" 2>> "$OUT/probe_k8.err"
RESHARD_K8_DIV=80 timeout 600 python scripts/probe_k8.py --fracs 0 > "$OUT/probe_k8_div80.jsonl" 2>> "$OUT/probe_k8.err"
timeout 600 python scripts/probe_k8.py --n 3000000 --fracs 0,20 > "$OUT/probe_k8_3m.jsonl" 2>> "$OUT/probe_k8.err"
echo done > "$OUT/DONE"
