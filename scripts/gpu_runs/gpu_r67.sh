#!/bin/bash
# r67: windowed K8 (bit-identity tests + window sweep vs the full-active-set variant;
# RESHARD_K8=full was retired after this run, so today the second pytest line runs the default)
set -u
OUT=gpurun_out/r67
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_dataset.py -m gpu -x -q -k "k8 or config5" > "$OUT/pytest_k8.log" 2>&1
RESHARD_K8=full timeout 600 python -m pytest tests/test_dataset.py -m gpu -x -q -k "k8" > "$OUT/pytest_k8_full.log" 2>&1
timeout 900 python scripts/probe_k8.py > "$OUT/probe_k8.jsonl" 2> "$OUT/probe_k8.err"
timeout 600 python scripts/probe_k8.py --n 3000000 > "$OUT/probe_k8_3m.jsonl" 2>> "$OUT/probe_k8.err"
echo done > "$OUT/DONE"
