#!/bin/bash
# round 2, call 60: fused K5 finalize compiled for 1 (64 regs), 5 (48) and 6 (40 regs + 8 B
# stack) resident blocks per SM; two repetitions; dataset tests on the chosen variant
O=gpurun_out/r2_60; mkdir -p $O
for rep in 1 2; do for m in 1 5 6; do
  RESHARD_K5_FIN_MINB=$m timeout 600 python bench.py --workload dataset-100m-dp2to4to8 --no-cpu-baseline --no-e2e > $O/m${m}_$rep.json 2> $O/m${m}_$rep.err
  python -c "import json;d=json.loads(open('$O/m${m}_$rep.json').read().strip().splitlines()[-1]);print('minb=$m rep=$rep',d['value'],d['roofline']['kernel_ms_per_step'],d['spot_check'])"
done; done
for m in 5 6; do RESHARD_K5_FIN_MINB=$m timeout 600 python -m pytest tests/test_dataset.py -m gpu -q -k batch > $O/pytest_m$m.txt 2>&1; tail -1 $O/pytest_m$m.txt; done
