#!/bin/bash
# round 2, call 25: SLOT claims for K3d (a claim = one grid-strided slot of a round of grid x K
# tiles, so concurrent tiles stay adjacent as in the static split) vs consecutive 8-tile claims
# vs static; parity of the slot kernel (executor suite forced onto it, stress)
O=gpurun_out/r2_25; mkdir -p $O
RESHARD_COPY_KERNEL=bulk_dyn RESHARD_DYN_SLOT=1 python -m pytest tests/test_gpu_executor.py tests/test_full_size.py -m gpu -q -x > $O/pytest_slot.txt 2>&1; tail -1 $O/pytest_slot.txt; grep -E "FAILED|rror" $O/pytest_slot.txt | head -5
RESHARD_DYN_SLOT=1 timeout 900 python scripts/stress_gpu.py --cases 800 > $O/stress_slot.txt 2>&1; tail -1 $O/stress_slot.txt
ab() { n=$1; shift; env "$@" timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-digests $W > $O/$n.json 2> $O/ab.err; python -c "import json;d=json.load(open('$O/$n.json'));print('$n',d['value'],d['ms_min'],d['roofline']['frac'],d['verify_mismatched_bytes'])"; }
for r in 1 2; do
for w in gpt2-small-tp2-to-pp2 gpt3-1.3b-dp-scaleout gpt3-6.7b-recovery gpt3-6.7b-tp4pp2-to-tp2pp2dp2; do
  W="--workload $w"
  ab ${w}_static_$r RESHARD_DYN_MIN_TILES=0
  ab ${w}_dyn8_$r RESHARD_COPY_KERNEL=bulk_dyn
  for c in 4 8 16; do ab ${w}_slot${c}_$r RESHARD_COPY_KERNEL=bulk_dyn RESHARD_DYN_SLOT=1 RESHARD_DYN_CLAIM=$c; done
done
done
