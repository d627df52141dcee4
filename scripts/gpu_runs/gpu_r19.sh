#!/bin/bash
# r19: dataset host-buffer e2e path — dataset GPU tests + dataset bench with e2e.
set -u
TAG=${1:-r19}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_dataset.py -m gpu -x -q > "$OUT/pytest_dataset.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_dataset.log"
timeout 900 python bench.py --workload dataset-100m-dp2to4to8 --steps 10 --warmup 3 > "$OUT/bench_dataset.json" 2> "$OUT/bench_dataset.err"
echo done > "$OUT/DONE"
