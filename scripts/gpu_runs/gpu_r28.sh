#!/bin/bash
set -u
TAG=${1:-r28}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
for b in 148 592 2368; do timeout 300 ./scripts/probe_pcie $b >> "$OUT/pcie.jsonl" 2>&1; done
echo done > "$OUT/DONE"
