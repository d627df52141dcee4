#!/bin/bash
# r53: fresh ncu --set full of the default workload's copy kernel on the final code path; bench
# lines of the wave workloads (traffic per wave launch).
set -u
OUT=gpurun_out/r53
mkdir -p "$OUT"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:copy_bulk -s 3 -c 1 \
  -o "$OUT/copy_default" python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > "$OUT/ncu.log" 2>&1
timeout 900 python bench.py --workload gpt3-6.7b-tp4pp2-to-tp2pp2dp2 --no-cpu-baseline > "$OUT/bench_67b.json" 2> "$OUT/bench.err"
timeout 600 python bench.py --workload gpt2-small-tp2-to-pp2 --no-cpu-baseline --no-e2e > "$OUT/bench_gpt2.json" 2>> "$OUT/bench.err"
echo done > "$OUT/DONE"
