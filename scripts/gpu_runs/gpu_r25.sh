#!/bin/bash
# r25: L2 evict_first hints on the bulk copies (RESHARD_BULK_HINT 0..3), same-box A/B on the
# default workload and GPT-3 6.7B waves.
set -u
TAG=${1:-r25}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 600 python -m pytest tests/test_gpu_executor.py -m gpu -x -q -k "fig6 or run_host" > "$OUT/pytest.log" 2>&1; echo "rc=$?" >> "$OUT/pytest.log"
: > "$OUT/ab.jsonl"
for rep in 1 2; do
for h in 0 1 2 3; do
  echo "{\"hint\": $h, \"rep\": $rep, \"w\": \"default\"}" >> "$OUT/ab.jsonl"
  RESHARD_BULK_HINT=$h timeout 300 python bench.py --no-cpu-baseline --no-e2e >> "$OUT/ab.jsonl" 2>> "$OUT/ab.err"
done
done
for h in 0 3; do
  echo "{\"hint\": $h, \"rep\": 1, \"w\": \"67b\"}" >> "$OUT/ab.jsonl"
  RESHARD_BULK_HINT=$h timeout 600 python bench.py --workload gpt3-6.7b-tp4pp2-to-tp2pp2dp2 --no-cpu-baseline >> "$OUT/ab.jsonl" 2>> "$OUT/ab.err"
done
echo done > "$OUT/DONE"
