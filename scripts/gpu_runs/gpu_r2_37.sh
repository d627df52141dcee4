#!/bin/bash
# round 2, call 37: ncu --set full of the fused K5 finalize pass; a long dataset stress run
O=gpurun_out/r2_37; mkdir -p $O
timeout 900 ncu --kernel-name regex:"repart_finalize2_multi" --launch-skip 3 --launch-count 1 --set full --clock-control none --import-source on \
  -o $O/k5_finalize python bench.py --workload dataset-100m-dp2to4to8 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/k5_finalize_ncu.out 2>&1; echo ncu rc=$?
timeout 2400 python scripts/stress_dataset.py --cases 4000 --seed 2037 > $O/stress_dataset.jsonl 2> $O/stress_dataset.err; tail -1 $O/stress_dataset.jsonl; tail -2 $O/stress_dataset.err
