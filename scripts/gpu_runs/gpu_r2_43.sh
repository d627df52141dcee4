#!/bin/bash
# round 2, call 43: bulk stage shape A/B on all four copy workloads (tiles are cut to the stage
# size, so the stage size sets how many rows of a fragment fit a tile): 7x29 (default), 6x32,
# 5x40, 4x48, 6x34, 7x30 KiB; default workload and GPT-2 small twice, the 6.7B ones once
O=gpurun_out/r2_43; mkdir -p $O
one() { tag=$1; w=$2; st=$3; kib=$4; shift 4; RESHARD_BULK_STAGES=$st RESHARD_BULK_STAGE_KIB=$kib timeout 900 python bench.py --workload $w --no-cpu-baseline --no-e2e --no-digests "$@" > $O/$tag.json 2> $O/$tag.err; python -c "import json;d=json.loads(open('$O/$tag.json').read().strip().splitlines()[-1]);print('$tag',d['value'],d['ms_min'],d['roofline']['frac'],d['verify_mismatched_bytes'],d['tiles'])" 2>&1 | tail -1; }
for rep in 1 2; do
  for sk in "7 29" "6 32" "5 40" "4 48" "6 34" "7 30"; do
    set -- $sk
    one gpt2_${1}x${2}_$rep gpt2-small-tp2-to-pp2 $1 $2
    one d13_${1}x${2}_$rep gpt3-1.3b-dp-scaleout $1 $2
  done
done
for sk in "7 29" "6 32" "5 40" "6 34"; do
  set -- $sk
  one cfg3_${1}x${2} gpt3-6.7b-tp4pp2-to-tp2pp2dp2 $1 $2 --steps 5 --warmup 3
  one cfg4_${1}x${2} gpt3-6.7b-recovery $1 $2 --steps 5 --warmup 3
done
