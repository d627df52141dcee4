#!/bin/bash
set -u
OUT=gpurun_out/r54
mkdir -p "$OUT"
timeout 300 ./scripts/probe_pcie 592 > "$OUT/pcie.jsonl" 2>&1
echo done > "$OUT/DONE"
