#!/bin/bash
set -u
TAG=${1:-r23b}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 1500 python -m pytest tests/test_dataset.py -m gpu -x -q > "$OUT/pytest_dataset.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_dataset.log"
timeout 300 python bench.py --workload dataset-100m-dp2to4to8 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > "$OUT/bench_dataset.json" 2>&1
W=gpt3-6.7b-tp4pp2-to-tp2pp2dp2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:copy_bulk -s 9 -c 1 \
  -o "$OUT/copy_67b" python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline > "$OUT/ncu_full.log" 2>&1
echo done > "$OUT/DONE"
