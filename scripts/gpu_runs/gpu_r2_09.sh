#!/bin/bash
# round 2, call 9: ncu --set full of the copy kernel on config 1 (0.94) and config 2 (1.02)
O=gpurun_out/r2_09; mkdir -p $O
for w in gpt2-small-tp2-to-pp2 gpt3-1.3b-dp-scaleout; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:copy_bulk_strided -s 3 -c 1 -o $O/full_$w python bench.py --workload $w --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_$w.out 2>&1; tail -1 $O/ncu_$w.out | cut -c1-200
done
