#!/bin/bash
# r34: consolidated evidence of the current tree — GPU suite, every workload's bench line,
# the reference arm, and the default workload's launch list.
set -u
TAG=${1:-r34}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 1800 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python __graft_entry__.py --smoke > "$OUT/smoke.log" 2>&1; echo "rc=$?" >> "$OUT/smoke.log"
timeout 600 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
timeout 900 python bench.py --impl reference > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
timeout 600 python bench.py --workload gpt2-small-tp2-to-pp2 > "$OUT/bench_gpt2.json" 2>> "$OUT/bench.err"
timeout 900 python bench.py --workload gpt3-6.7b-tp4pp2-to-tp2pp2dp2 --no-cpu-baseline > "$OUT/bench_67b.json" 2>> "$OUT/bench.err"
timeout 900 python bench.py --workload gpt3-6.7b-recovery --no-cpu-baseline > "$OUT/bench_67b_recovery.json" 2>> "$OUT/bench.err"
timeout 900 python bench.py --workload dataset-100m-dp2to4to8 --steps 10 --warmup 3 > "$OUT/bench_dataset.json" 2>> "$OUT/bench.err"
timeout 600 python bench.py --workload gpt3-1.3b-dp-scaleout --mode central --no-cpu-baseline > "$OUT/bench_central.json" 2>> "$OUT/bench.err"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file "$OUT/launches.csv" \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > "$OUT/ncu_launches.log" 2>&1
echo done > "$OUT/DONE"
