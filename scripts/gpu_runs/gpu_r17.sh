#!/bin/bash
# r17: K5 split2 default — GPU suite, default + dataset bench, dataset launch list, ncu of the gather pass.
set -u
TAG=${1:-r17}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 1500 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_gpu.log"
timeout 600 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
timeout 900 python bench.py --workload dataset-100m-dp2to4to8 --steps 10 --warmup 3 > "$OUT/bench_dataset.json" 2> "$OUT/bench_dataset.err"
RESHARD_K5=lookback timeout 900 python bench.py --workload dataset-100m-dp2to4to8 --steps 10 --warmup 3 --no-cpu-baseline > "$OUT/bench_dataset_lookback.json" 2>> "$OUT/bench_dataset.err"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"repart|probe" \
  --csv --log-file "$OUT/launches_dataset.csv" python bench.py --workload dataset-100m-dp2to4to8 --steps 3 --warmup 3 --no-cpu-baseline > "$OUT/ncu_launches.log" 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:repart_gather2 -s 12 -c 1 \
  -o "$OUT/gather2" python bench.py --workload dataset-100m-dp2to4to8 --steps 1 --warmup 3 --no-cpu-baseline > "$OUT/ncu_full.log" 2>&1
echo done > "$OUT/DONE"
