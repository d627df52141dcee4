#!/bin/bash
# round 2, call 20: ncu --set full of the new default long-launch kernel (bulk_dyn) per workload,
# and the default workload's launch list
O=gpurun_out/r2_20; mkdir -p $O
for w in gpt3-1.3b-dp-scaleout gpt3-6.7b-tp4pp2-to-tp2pp2dp2 gpt3-6.7b-recovery; do
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:copy_bulk_dyn -s 3 -c 1 -o $O/full_$w python bench.py --workload $w --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-digests > $O/ncu_$w.out 2>&1; tail -1 $O/ncu_$w.out | cut -c1-150
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-digests > $O/launches.out 2>&1; echo launches rc=$?
