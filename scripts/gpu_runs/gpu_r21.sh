#!/bin/bash
set -u
TAG=${1:-r21}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"repart_finalize2|repart_tile_scan" -s 24 -c 2 \
  -o "$OUT/finalize" python bench.py --workload dataset-100m-dp2to4to8 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > "$OUT/ncu_full.log" 2>&1
echo done > "$OUT/DONE"
