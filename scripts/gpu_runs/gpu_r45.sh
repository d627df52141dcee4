#!/bin/bash
set -u
OUT=gpurun_out/r45
mkdir -p "$OUT"
timeout 300 python __graft_entry__.py --smoke > "$OUT/smoke.log" 2>&1; echo "rc=$?" >> "$OUT/smoke.log"
timeout 600 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
echo done > "$OUT/DONE"
