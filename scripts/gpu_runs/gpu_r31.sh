#!/bin/bash
# r31: ncu --set full of the copy kernel on GPT-2 small (config 1) and GPT-3 6.7B recovery
# (config 4, one wave), plus the GPU suite on the reverted K8.
set -u
TAG=${1:-r31}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 1800 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_gpu.log"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:copy_bulk -s 3 -c 1 \
  -o "$OUT/copy_gpt2" python bench.py --workload gpt2-small-tp2-to-pp2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > "$OUT/ncu_gpt2.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:copy_bulk -s 6 -c 1 \
  -o "$OUT/copy_recovery" python bench.py --workload gpt3-6.7b-recovery --steps 1 --warmup 3 --no-cpu-baseline > "$OUT/ncu_recovery.log" 2>&1
echo done > "$OUT/DONE"
