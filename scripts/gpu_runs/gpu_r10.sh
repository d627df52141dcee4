#!/bin/bash
set -u
TAG=${1:-r10}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
RESHARD_COPY_KERNEL=bulk_warp timeout 900 python -m pytest tests/test_gpu_executor.py -m gpu -x -q > "$OUT/pytest_warp.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_warp.log"
timeout 900 python -m pytest tests/test_gpu_multiprocess.py -m gpu -x -q > "$OUT/pytest_mp.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_mp.log"
B="python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline"
: > "$OUT/ab.jsonl"
for k in bulk_strided bulk_warp; do
  for w in gpt3-1.3b-dp-scaleout gpt2-small-tp2-to-pp2; do
    echo "{\"env\": \"$k\", \"workload\": \"$w\"}" >> "$OUT/ab.jsonl"
    RESHARD_COPY_KERNEL=$k timeout 300 $B --workload $w >> "$OUT/ab.jsonl" 2>> "$OUT/ab.err"
  done
  echo "{\"env\": \"$k\", \"workload\": \"67b\"}" >> "$OUT/ab.jsonl"
  RESHARD_COPY_KERNEL=$k timeout 900 python bench.py --workload gpt3-6.7b-tp4pp2-to-tp2pp2dp2 --steps 3 --warmup 3 --no-cpu-baseline >> "$OUT/ab.jsonl" 2>> "$OUT/ab.err"
done
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
echo done > "$OUT/DONE"
