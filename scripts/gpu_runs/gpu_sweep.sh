#!/bin/bash
# Kernel-variant sweep + tests on the B200 box.  Usage: gpurun -- 'bash scripts/gpu_sweep.sh <tag>'
set -u
TAG=${1:-sweep}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
B="python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline"

timeout 900 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu_ldg.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_gpu_ldg.log"
RESHARD_COPY_KERNEL=bulk timeout 900 python -m pytest tests/test_gpu_executor.py -m gpu -x -q > "$OUT/pytest_gpu_bulk.log" 2>&1
echo "rc=$?" >> "$OUT/pytest_gpu_bulk.log"

: > "$OUT/sweep.jsonl"
run() {  # env..., then tile
  local tile=$1; shift
  echo "{\"env\": \"$*\", \"tile_kib\": $tile}" >> "$OUT/sweep.jsonl"
  env "$@" timeout 300 $B --tile-kib "$tile" >> "$OUT/sweep.jsonl" 2>> "$OUT/sweep.err"
}
for tile in 128 256 1024; do
  for c in 2 3; do run $tile RESHARD_COPY_KERNEL=ldg RESHARD_CTAS_PER_SM=$c; done
  run $tile RESHARD_COPY_KERNEL=ldg8 RESHARD_CTAS_PER_SM=2
done
for sv in "6 32" "8 24" "4 48" "12 16" "3 64"; do
  set -- $sv
  run 256 RESHARD_COPY_KERNEL=bulk RESHARD_CTAS_PER_SM=1 RESHARD_BULK_STAGES=$1 RESHARD_BULK_STAGE_KIB=$2
done
run 256 RESHARD_COPY_KERNEL=bulk RESHARD_CTAS_PER_SM=2 RESHARD_BULK_STAGES=6 RESHARD_BULK_STAGE_KIB=16
run 256 RESHARD_COPY_KERNEL=bulk RESHARD_CTAS_PER_SM=2 RESHARD_BULK_STAGES=4 RESHARD_BULK_STAGE_KIB=24
# other workloads with the default kernel
timeout 600 python bench.py --workload gpt2-small-tp2-to-pp2 --steps 20 --warmup 5 > "$OUT/bench_gpt2.json" 2>&1
timeout 900 python bench.py --workload dataset-100m-dp2to4to8 --steps 10 --warmup 3 > "$OUT/bench_dataset.json" 2>&1
# ncu: bulk kernel and dataset kernel, one launch each
RESHARD_COPY_KERNEL=bulk timeout 900 ncu --set full --clock-control none --import-source on -k regex:copy_bulk -s 3 -c 1 \
  -o "$OUT/copy_bulk" $B --steps 3 --warmup 3 > "$OUT/ncu_bulk.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:copy_v16 -s 3 -c 1 \
  -o "$OUT/copy_v16" $B --steps 3 --warmup 3 > "$OUT/ncu_v16.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:repartition -s 4 -c 1 \
  -o "$OUT/repartition" python bench.py --workload dataset-100m-dp2to4to8 --steps 1 --warmup 3 --no-cpu-baseline \
  > "$OUT/ncu_dataset.log" 2>&1
echo done > "$OUT/DONE"
