#!/bin/bash
# round 2, call 33: K5 batch with stream priorities (gathers high, scan + finalize low) vs equal
# priorities vs per-rank calls, two repetitions; parity of the batch test
O=gpurun_out/r2_33; mkdir -p $O
timeout 900 python -m pytest tests/test_dataset.py -m gpu -q -k batch > $O/pytest_batch.txt 2>&1; tail -1 $O/pytest_batch.txt
run() { n=$1; shift; timeout 1200 python bench.py "$@" > $O/$n.json 2> $O/$n.err || echo "$n rc=$?"; python -c "import json;d=json.loads(open('$O/$n.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$n',d.get('value'),r['kernel_ms_per_step'],r['gather_write_floor_ms'],r['step_frac_of_floor'],d['spot_check'])" 2>&1 | tail -1; }
for rep in 1 2; do
  run prio_$rep --workload dataset-100m-dp2to4to8 --no-cpu-baseline --no-e2e
  RESHARD_K5_PRIO=0 run noprio_$rep --workload dataset-100m-dp2to4to8 --no-cpu-baseline --no-e2e
  RESHARD_K5_BATCH=0 run perrank_$rep --workload dataset-100m-dp2to4to8 --no-cpu-baseline --no-e2e
done
