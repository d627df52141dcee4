#!/bin/bash
# round 2, call 40: fused K5 finalize tiles-per-block sweep (1, 2, 4, 8, 16), two repetitions
O=gpurun_out/r2_40; mkdir -p $O
for rep in 1 2; do for ft in 1 2 4 8 16; do
  RESHARD_K5_FIN_TILES=$ft timeout 600 python bench.py --workload dataset-100m-dp2to4to8 --no-cpu-baseline --no-e2e > $O/ft${ft}_$rep.json 2> $O/ft${ft}_$rep.err
  python -c "import json;d=json.loads(open('$O/ft${ft}_$rep.json').read().strip().splitlines()[-1]);print('ft=$ft rep=$rep',d['value'],d['roofline']['kernel_ms_per_step'],d['spot_check'])"
done; done
