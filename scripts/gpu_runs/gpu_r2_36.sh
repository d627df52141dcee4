#!/bin/bash
# round 2, call 36: dataset GPU tests after the fused-path fallback fix; dataset stress run incl.
# the multi-rank batches; launch list of the dataset step's K5 kernels
O=gpurun_out/r2_36; mkdir -p $O
timeout 900 python -m pytest tests/test_dataset.py -m gpu -q > $O/pytest_dataset.txt 2>&1; tail -1 $O/pytest_dataset.txt
timeout 900 ncu --kernel-name regex:"repart" --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_k5.csv python bench.py --workload dataset-100m-dp2to4to8 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/launches_k5.out 2>&1; echo launches_k5 rc=$?
timeout 2400 python scripts/stress_dataset.py --cases 400 --seed 2036 > $O/stress_dataset.jsonl 2> $O/stress_dataset.err; tail -1 $O/stress_dataset.jsonl; tail -2 $O/stress_dataset.err
