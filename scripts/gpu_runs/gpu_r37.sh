#!/bin/bash
# r37: host-buffer pipeline with ramped chunk sizes — GPT-2 small and the default workload.
set -u
OUT=gpurun_out/r37
mkdir -p "$OUT"
timeout 600 python -m pytest tests/test_gpu_executor.py -m gpu -x -q -k run_host > "$OUT/pytest.log" 2>&1; echo "rc=$?" >> "$OUT/pytest.log"
for cfg in "64 0" "16 16" "16 32" "8 32" "32 16"; do
  set -- $cfg
  echo "{\"chunks\": $1, \"ramp\": $2}" >> "$OUT/gpt2.jsonl"
  RESHARD_HOST_CHUNKS=$1 RESHARD_HOST_RAMP=$2 timeout 300 python bench.py --workload gpt2-small-tp2-to-pp2 --no-cpu-baseline --e2e-steps 5 >> "$OUT/gpt2.jsonl" 2>> "$OUT/err"
done
for cfg in "64 0" "16 16" "16 32"; do
  set -- $cfg
  echo "{\"chunks\": $1, \"ramp\": $2}" >> "$OUT/default.jsonl"
  RESHARD_HOST_CHUNKS=$1 RESHARD_HOST_RAMP=$2 timeout 300 python bench.py --no-cpu-baseline --e2e-steps 3 >> "$OUT/default.jsonl" 2>> "$OUT/err"
done
echo done > "$OUT/DONE"
