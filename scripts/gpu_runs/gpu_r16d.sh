#!/bin/bash
# r16d: gather-only vs gather+write floor probes, L2 fetch granularity 0/32/64/128.
set -u
TAG=${1:-r16d}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
: > "$OUT/probe.jsonl"
for pr in read write; do
for l2 in 0 32 64 128; do
  echo "{\"probe\": \"$pr\", \"l2\": $l2}" >> "$OUT/probe.jsonl"
  RESHARD_PROBE=$pr RESHARD_L2_FETCH=$l2 timeout 300 python bench.py --workload dataset-100m-dp2to4to8 --steps 5 --warmup 3 --no-cpu-baseline >> "$OUT/probe.jsonl" 2>> "$OUT/probe.err"
done
done
for l2 in 0 32; do
RESHARD_L2_FETCH=$l2 RESHARD_PROBE=write timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:"probe|repartition" \
  --csv --log-file "$OUT/launches_l2_$l2.csv" python bench.py --workload dataset-100m-dp2to4to8 --steps 3 --warmup 3 --no-cpu-baseline > "$OUT/ncu_$l2.log" 2>&1
done
echo done > "$OUT/DONE"
