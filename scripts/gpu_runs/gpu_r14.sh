#!/bin/bash
# r14: GPU suite (central mode, reference fixtures on device), default bench, central-mode
# bench, dataset bench with the random-gather floor.  Usage: gpurun -- 'bash scripts/gpu_runs/gpu_r14.sh'
set -u
TAG=${1:-r14}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 1500 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_gpu.log"
timeout 600 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
for w in gpt3-1.3b-dp-scaleout gpt2-small-tp2-to-pp2; do
  timeout 600 python bench.py --workload $w --mode central --no-cpu-baseline > "$OUT/bench_central_$w.json" 2>> "$OUT/bench_central.err"
done
timeout 600 python bench.py --workload gpt2-small-tp2-to-pp2 --no-cpu-baseline > "$OUT/bench_gpt2.json" 2>> "$OUT/bench_gpt2.err"
timeout 900 python bench.py --workload dataset-100m-dp2to4to8 --steps 10 --warmup 3 > "$OUT/bench_dataset.json" 2> "$OUT/bench_dataset.err"
echo done > "$OUT/DONE"
