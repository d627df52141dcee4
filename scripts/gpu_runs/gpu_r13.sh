#!/bin/bash
# r13: GPU suite (incl. full-size config 5 parity), bench with the PCIe probe, host-chunk
# sweep of the e2e pipeline, K5 register/occupancy A/B.  Usage: gpurun -- 'bash scripts/gpu_runs/gpu_r13.sh'
set -u
TAG=${1:-r13}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 1500 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_gpu.log"
timeout 600 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
: > "$OUT/host_chunks.jsonl"
for c in 8 16 64 128; do
  echo "{\"host_chunks\": $c}" >> "$OUT/host_chunks.jsonl"
  RESHARD_HOST_CHUNKS=$c timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 >> "$OUT/host_chunks.jsonl" 2>> "$OUT/host_chunks.err"
done
: > "$OUT/k5.jsonl"
for rep in 1 2; do
for m in lookback lookback4 split; do
  echo "{\"k5\": \"$m\", \"rep\": $rep}" >> "$OUT/k5.jsonl"
  RESHARD_K5=$m timeout 900 python bench.py --workload dataset-100m-dp2to4to8 --steps 10 --warmup 3 --no-cpu-baseline >> "$OUT/k5.jsonl" 2>> "$OUT/k5.err"
done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:repartition_kernel -s 12 -c 1 \
  -o "$OUT/repart" python bench.py --workload dataset-100m-dp2to4to8 --steps 1 --warmup 3 --no-cpu-baseline \
  > "$OUT/ncu_dataset.log" 2>&1
echo done > "$OUT/DONE"
