#!/bin/bash
# round 2, call 34: K5 fused batch (one launch per pass for all ranks of a GPU) vs the
# two-stream batch vs per-rank calls; parity, memcheck / racecheck of the fused path
O=gpurun_out/r2_34; mkdir -p $O
timeout 900 python -m pytest tests/test_dataset.py -m gpu -q > $O/pytest_dataset.txt 2>&1; tail -1 $O/pytest_dataset.txt; grep FAILED $O/pytest_dataset.txt | head
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_dataset.py -m gpu -q -k "batch and 32-True" > $O/memcheck_fused.txt 2>&1; tail -2 $O/memcheck_fused.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_dataset.py -m gpu -q -k "batch and 32-True" > $O/racecheck_fused.txt 2>&1; tail -2 $O/racecheck_fused.txt
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_dataset.py -m gpu -q -k "batch and 32-True" > $O/synccheck_fused.txt 2>&1; tail -2 $O/synccheck_fused.txt
run() { n=$1; shift; timeout 1200 python bench.py "$@" > $O/$n.json 2> $O/$n.err || echo "$n rc=$?"; python -c "import json;d=json.loads(open('$O/$n.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$n',d.get('value'),r['kernel_ms_per_step'],r['gather_write_floor_ms'],r['step_frac_of_floor'],r['frac'],d['spot_check'])" 2>&1 | tail -1; }
for rep in 1 2; do
  run fused_$rep --workload dataset-100m-dp2to4to8 --no-cpu-baseline --no-e2e
  RESHARD_K5_FUSE=0 run streams_$rep --workload dataset-100m-dp2to4to8 --no-cpu-baseline --no-e2e
  RESHARD_K5_BATCH=0 run perrank_$rep --workload dataset-100m-dp2to4to8 --no-cpu-baseline --no-e2e
done
