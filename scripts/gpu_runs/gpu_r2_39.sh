#!/bin/bash
# round 2, call 39: fused K5 finalize software-pipelined over 4 tiles per block (double-buffered
# warp totals) — parity, sanitizers, stress, step time, launch list
O=gpurun_out/r2_39; mkdir -p $O
timeout 900 python -m pytest tests/test_dataset.py -m gpu -q > $O/pytest_dataset.txt 2>&1; tail -1 $O/pytest_dataset.txt; grep FAILED $O/pytest_dataset.txt | head -3
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_dataset.py -m gpu -q -k "batch and 32-True" > $O/${tool}_fused.txt 2>&1; tail -2 $O/${tool}_fused.txt | head -1
done
timeout 1200 python scripts/stress_dataset.py --cases 1000 --seed 2039 > $O/stress_dataset.jsonl 2> $O/stress_dataset.err; tail -1 $O/stress_dataset.jsonl; tail -2 $O/stress_dataset.err
run() { n=$1; shift; timeout 1200 python bench.py "$@" > $O/$n.json 2> $O/$n.err || echo "$n rc=$?"; python -c "import json;d=json.loads(open('$O/$n.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$n',d.get('value'),r['kernel_ms_per_step'],r['frac'],d['spot_check'])" 2>&1 | tail -1; }
for rep in 1 2; do run fused_$rep --workload dataset-100m-dp2to4to8 --no-cpu-baseline --no-e2e; done
timeout 900 ncu --kernel-name regex:"repart" --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -c 60 --csv --log-file $O/launches_k5.csv python bench.py --workload dataset-100m-dp2to4to8 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/launches_k5.out 2>&1; echo launches_k5 rc=$?
