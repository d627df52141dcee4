#!/bin/bash
set -u
OUT=gpurun_out/r51
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_gpu_executor.py -m gpu -x -q -k broadcast > "$OUT/pytest.log" 2>&1; echo "rc=$?" >> "$OUT/pytest.log"
timeout 600 python scripts/probe_broadcast.py > "$OUT/broadcast.jsonl" 2>&1
echo done > "$OUT/DONE"
