#!/bin/bash
set -u
OUT=gpurun_out/r61b
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_checkpoint.py -m gpu -x -q > "$OUT/pytest.log" 2>&1; echo "rc=$?" >> "$OUT/pytest.log"
for t in 1 8 16; do RESHARD_IO_THREADS=$t timeout 900 python scripts/probe_checkpoint.py | sed "s/^{/{\"threads\": $t, /" >> "$OUT/checkpoint.jsonl" 2>&1; done
echo done > "$OUT/DONE"
