#!/bin/bash
# r43: GPU stress run of the data plane vs the oracle (scripts/stress_gpu.py).
set -u
OUT=gpurun_out/r43
mkdir -p "$OUT"
timeout 2400 python scripts/stress_gpu.py --cases 3000 > "$OUT/stress.jsonl" 2> "$OUT/stress.err"; timeout 2400 python scripts/stress_gpu.py --cases 30000 --seed 7 > "$OUT/stress_30k.jsonl" 2> "$OUT/stress.err"; echo "rc=$?" >> "$OUT/stress.err"
echo done > "$OUT/DONE"
