#!/bin/bash
# round 2, call 42: GPT-2 small (the shortest copy launch, 0.94 of HBM) — CTAs per SM x stages x
# stage size, and the dynamic-claim kernel with small claims; two repetitions of each
O=gpurun_out/r2_42; mkdir -p $O
one() { tag=$1; shift; env "$@" timeout 300 python bench.py --workload gpt2-small-tp2-to-pp2 --no-cpu-baseline --no-e2e --no-digests > $O/$tag.json 2> $O/$tag.err; python -c "import json;d=json.loads(open('$O/$tag.json').read().strip().splitlines()[-1]);print('$tag',d['value'],d['ms_min'],d['roofline']['frac'],d['verify_mismatched_bytes'])" 2>&1 | tail -1; }
for rep in 1 2; do
  one base_$rep X=1
  one c1s8k24_$rep RESHARD_BULK_STAGES=8 RESHARD_BULK_STAGE_KIB=24
  one c1s6k32_$rep RESHARD_BULK_STAGES=6 RESHARD_BULK_STAGE_KIB=32
  one c1s12k16_$rep RESHARD_BULK_STAGES=12 RESHARD_BULK_STAGE_KIB=16
  one c2s4k24_$rep RESHARD_CTAS_PER_SM=2 RESHARD_BULK_STAGES=4 RESHARD_BULK_STAGE_KIB=24
  one c2s3k32_$rep RESHARD_CTAS_PER_SM=2 RESHARD_BULK_STAGES=3 RESHARD_BULK_STAGE_KIB=32
  one c2s6k16_$rep RESHARD_CTAS_PER_SM=2 RESHARD_BULK_STAGES=6 RESHARD_BULK_STAGE_KIB=16
  one c3s4k16_$rep RESHARD_CTAS_PER_SM=3 RESHARD_BULK_STAGES=4 RESHARD_BULK_STAGE_KIB=16
  one dyn2_$rep RESHARD_COPY_KERNEL=bulk_dyn RESHARD_DYN_CLAIM=2
  one dyn4_$rep RESHARD_COPY_KERNEL=bulk_dyn RESHARD_DYN_CLAIM=4
done
