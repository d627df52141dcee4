#!/bin/bash
# r20: sanitizers over the new K5 kernels (split2 gather / tile scan / finalize, index pad,
# host-buffer path), plus the ncu --set full capture of the padded gather pass.
set -u
TAG=${1:-r20}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
S=/usr/local/cuda/bin/compute-sanitizer
timeout 1800 $S --tool memcheck --error-exitcode 9 python -m pytest tests/test_dataset.py -m gpu -x -q > "$OUT/memcheck_dataset.log" 2>&1; echo "rc=$?" >> "$OUT/memcheck_dataset.log"
timeout 1800 $S --tool racecheck --error-exitcode 9 python -m pytest tests/test_dataset.py -m gpu -x -q -k "k5 or host_buffer" > "$OUT/racecheck_dataset.log" 2>&1; echo "rc=$?" >> "$OUT/racecheck_dataset.log"
timeout 1800 $S --tool synccheck --error-exitcode 9 python -m pytest tests/test_dataset.py -m gpu -x -q -k "k5" > "$OUT/synccheck_dataset.log" 2>&1; echo "rc=$?" >> "$OUT/synccheck_dataset.log"
timeout 1200 $S --tool memcheck --error-exitcode 9 python __graft_entry__.py --smoke > "$OUT/memcheck_smoke.log" 2>&1; echo "rc=$?" >> "$OUT/memcheck_smoke.log"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:repart_gather2 -s 12 -c 1 \
  -o "$OUT/gather2_padded" python bench.py --workload dataset-100m-dp2to4to8 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > "$OUT/ncu_full.log" 2>&1
echo done > "$OUT/DONE"
