#!/bin/bash
# Round-1 check #5: fan-out tiles, 7x29 default, dataset L2 fetch granularity sweep.
set -u
TAG=${1:-r05}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 600 python __graft_entry__.py --smoke > "$OUT/smoke.log" 2>&1; echo "rc=$?" >> "$OUT/smoke.log"
timeout 1200 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_gpu.log"
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
timeout 1800 python bench.py --workload gpt3-6.7b-tp4pp2-to-tp2pp2dp2 --steps 3 --warmup 3 --no-cpu-baseline > "$OUT/bench_67b.json" 2> "$OUT/bench_67b.err"
RESHARD_FANOUT=0 timeout 1800 python bench.py --workload gpt3-6.7b-tp4pp2-to-tp2pp2dp2 --steps 3 --warmup 3 --no-cpu-baseline > "$OUT/bench_67b_nofan.json" 2> "$OUT/bench_67b_nofan.err"
timeout 900 python bench.py --workload gpt2-small-tp2-to-pp2 --steps 20 --warmup 5 > "$OUT/bench_gpt2.json" 2>&1
for g in 32 64 128 0; do
  RESHARD_L2_FETCH=$g timeout 900 python bench.py --workload dataset-100m-dp2to4to8 --steps 10 --warmup 3 --no-cpu-baseline > "$OUT/bench_dataset_l2_$g.json" 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > "$OUT/ncu_launch.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:copy_bulk -s 3 -c 1 \
  -o "$OUT/copy_bulk" python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > "$OUT/ncu_bulk.log" 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:copy_bulk -s 9 -c 1 \
  -o "$OUT/copy_bulk_67b" python bench.py --workload gpt3-6.7b-tp4pp2-to-tp2pp2dp2 --steps 1 --warmup 3 --no-cpu-baseline > "$OUT/ncu_bulk_67b.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:repartition -s 4 -c 1 \
  -o "$OUT/repartition" python bench.py --workload dataset-100m-dp2to4to8 --steps 1 --warmup 3 --no-cpu-baseline \
  > "$OUT/ncu_dataset.log" 2>&1
echo done > "$OUT/DONE"
