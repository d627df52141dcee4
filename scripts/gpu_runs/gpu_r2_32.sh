#!/bin/bash
# round 2, call 32: K5 batch (several ranks per GPU: gather passes back to back, scan + finalize
# on a second stream) — parity tests, memcheck of the batch test, dataset line A/B (batch vs per rank) x2
O=gpurun_out/r2_32; mkdir -p $O
timeout 900 python -m pytest tests/test_dataset.py -m gpu -q > $O/pytest_dataset.txt 2>&1; tail -2 $O/pytest_dataset.txt; grep FAILED $O/pytest_dataset.txt | head
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_dataset.py -m gpu -q -k "batch and 32" > $O/memcheck_batch.txt 2>&1; tail -3 $O/memcheck_batch.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_dataset.py -m gpu -q -k "batch and 32" > $O/racecheck_batch.txt 2>&1; tail -3 $O/racecheck_batch.txt
run() { n=$1; shift; timeout 1200 python bench.py "$@" > $O/$n.json 2> $O/$n.err || echo "$n rc=$?"; python -c "import json;d=json.loads(open('$O/$n.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$n',d.get('value'),r['kernel_ms_per_step'],r['gather_write_floor_ms'],r['step_frac_of_floor'],d['spot_check'],(d.get('e2e') or {}).get('value'))" 2>&1 | tail -1; }
for rep in 1 2; do
  run batch_$rep --workload dataset-100m-dp2to4to8 --no-cpu-baseline --no-e2e
  RESHARD_K5_BATCH=0 run perrank_$rep --workload dataset-100m-dp2to4to8 --no-cpu-baseline --no-e2e
done
