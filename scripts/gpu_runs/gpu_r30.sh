#!/bin/bash
# r30: K8 in one cooperative launch vs two launches per round — parity + same-box A/B; NVTX build smoke.
set -u
export PYTHONPATH=$PWD
TAG=${1:-r30}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_dataset.py -m gpu -x -q > "$OUT/pytest_dataset.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_dataset.log"
cat > "$OUT/k8.py" <<'PY'
import os, statistics
import numpy as np
import paper_2312_05181_b200 as rs
ctx = rs.Context(1, [0], [0])
n = 100_000_000
p = ctx.malloc(0, 8 * n)
ms = [rs.shuffle_epoch_device(ctx, 0, n, 0x5EED, 0, p) for _ in range(6)]
print({"k8": os.environ.get("RESHARD_K8", "coop"), "ms": [round(t["ms"], 3) for t in ms], "mean_last5": round(statistics.mean(t["ms"] for t in ms[1:]), 3),
       "rounds": ms[-1]["rounds"], "launches": ms[-1]["launches"]})
PY
for rep in 1 2; do
  RESHARD_K8=rounds timeout 300 python "$OUT/k8.py" >> "$OUT/k8.txt" 2>&1
  timeout 300 python "$OUT/k8.py" >> "$OUT/k8.txt" 2>&1
done
echo done > "$OUT/DONE"
