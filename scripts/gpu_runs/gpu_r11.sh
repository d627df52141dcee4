#!/bin/bash
set -u
TAG=${1:-r11}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
for m in split lookback; do
  RESHARD_K5=$m timeout 900 python bench.py --workload dataset-100m-dp2to4to8 --steps 10 --warmup 3 --no-cpu-baseline > "$OUT/bench_dataset_$m.json" 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:repart -s 12 -c 3 \
  -o "$OUT/repart_split" python bench.py --workload dataset-100m-dp2to4to8 --steps 1 --warmup 3 --no-cpu-baseline \
  > "$OUT/ncu_dataset.log" 2>&1
# sanitizers on small cases (memcheck: device memory errors; racecheck/synccheck: shared memory / barriers)
S=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $S --tool memcheck --error-exitcode 9 python __graft_entry__.py --smoke > "$OUT/memcheck_smoke.log" 2>&1; echo "rc=$?" >> "$OUT/memcheck_smoke.log"
timeout 1800 $S --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_executor.py -m gpu -x -q -k "fig6 or recovery or merge_error or run_host" > "$OUT/memcheck_executor.log" 2>&1; echo "rc=$?" >> "$OUT/memcheck_executor.log"
timeout 1800 $S --tool memcheck --error-exitcode 9 python -m pytest tests/test_dataset.py -m gpu -x -q > "$OUT/memcheck_dataset.log" 2>&1; echo "rc=$?" >> "$OUT/memcheck_dataset.log"
timeout 1800 $S --tool racecheck --error-exitcode 9 python -m pytest tests/test_dataset.py -m gpu -x -q -k k5 > "$OUT/racecheck_dataset.log" 2>&1; echo "rc=$?" >> "$OUT/racecheck_dataset.log"
timeout 1800 $S --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_executor.py -m gpu -x -q -k "fig6 or recovery" > "$OUT/synccheck_executor.log" 2>&1; echo "rc=$?" >> "$OUT/synccheck_executor.log"
echo done > "$OUT/DONE"
