#!/bin/bash
# round 2, call 38: fused K5 with the rank table as a by-value kernel parameter (constant bank)
# and the finalize's tile prefix load hoisted — parity, stress (chunks of <= 16 ranks), A/B, ncu
O=gpurun_out/r2_38; mkdir -p $O
timeout 900 python -m pytest tests/test_dataset.py -m gpu -q > $O/pytest_dataset.txt 2>&1; tail -1 $O/pytest_dataset.txt; grep FAILED $O/pytest_dataset.txt | head -3
timeout 1200 python scripts/stress_dataset.py --cases 1000 --seed 2038 > $O/stress_dataset.jsonl 2> $O/stress_dataset.err; tail -1 $O/stress_dataset.jsonl; tail -2 $O/stress_dataset.err
run() { n=$1; shift; timeout 1200 python bench.py "$@" > $O/$n.json 2> $O/$n.err || echo "$n rc=$?"; python -c "import json;d=json.loads(open('$O/$n.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$n',d.get('value'),r['kernel_ms_per_step'],r['frac'],d['spot_check'])" 2>&1 | tail -1; }
for rep in 1 2; do
  run fused_$rep --workload dataset-100m-dp2to4to8 --no-cpu-baseline --no-e2e
done
timeout 900 ncu --kernel-name regex:"repart" --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_k5.csv python bench.py --workload dataset-100m-dp2to4to8 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/launches_k5.out 2>&1; echo launches_k5 rc=$?
timeout 900 ncu --kernel-name regex:"repart_finalize2_multi" --launch-skip 3 --launch-count 1 --set full --clock-control none --import-source on \
  -o $O/k5_finalize python bench.py --workload dataset-100m-dp2to4to8 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/k5_finalize_ncu.out 2>&1; echo ncu rc=$?
