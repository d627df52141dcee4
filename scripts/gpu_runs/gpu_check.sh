#!/bin/bash
# One GPU round on the B200 box: smoke, GPU tests, bench, ncu launch list + full capture.
# Usage (from the container):  gpurun --timeout 2400 -- 'bash scripts/gpu_check.sh [tag]'
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
{
  echo "== host"; nproc; lscpu | grep -E "Model name|Socket|Thread|NUMA node\(s\)"; free -g | head -2
  nvidia-smi --query-gpu=name,memory.total,clocks.max.sm,power.limit --format=csv
} > "$OUT/host.txt" 2>&1

timeout 600 python __graft_entry__.py --smoke > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log"
timeout 1500 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?" >> "$OUT/bench.err"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
# every launch with its device time (shares, not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > "$OUT/ncu_launch_bench.log" 2>&1
# the top kernel, full set, one launch after warm-up
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:copy_tiles -s 3 -c 1 \
  -o "$OUT/copy_tiles" python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > "$OUT/ncu_full.log" 2>&1
echo done > "$OUT/DONE"
