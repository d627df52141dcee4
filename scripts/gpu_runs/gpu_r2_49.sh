#!/bin/bash
# round 2, call 49: larger power-of-two stages (3 x 64 KiB) and 2 CTAs/SM x 3 x 32 KiB vs the
# 6 x 32 KiB default, on GPT-2 small, 1.3B and the recovery; two repetitions
O=gpurun_out/r2_49; mkdir -p $O
one() { tag=$1; w=$2; shift 2; env "$@" timeout 900 python bench.py --workload $w --no-cpu-baseline --no-e2e --no-digests --steps 10 > $O/$tag.json 2> $O/$tag.err; python -c "import json;d=json.loads(open('$O/$tag.json').read().strip().splitlines()[-1]);print('$tag',d['value'],d['ms_min'],d['roofline']['frac'],d['verify_mismatched_bytes'],d['tiles'])" 2>&1 | tail -1; }
for rep in 1 2; do
  for w in gpt2-small-tp2-to-pp2 gpt3-1.3b-dp-scaleout gpt3-6.7b-recovery; do
    one ${w}_6x32_$rep $w X=1
    one ${w}_3x64_$rep $w RESHARD_BULK_STAGES=3 RESHARD_BULK_STAGE_KIB=64
    one ${w}_c2_3x32_$rep $w RESHARD_CTAS_PER_SM=2 RESHARD_BULK_STAGES=3 RESHARD_BULK_STAGE_KIB=32
  done
done
