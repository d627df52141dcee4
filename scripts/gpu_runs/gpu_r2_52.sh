#!/bin/bash
# round 2, call 52: K3T tensor-map boxes re-checked at 32 KiB stages (GPT-2 small, 1.3B, 6.7B)
O=gpurun_out/r2_52; mkdir -p $O
one() { tag=$1; w=$2; e=$3; shift 3; env $e timeout 900 python bench.py --workload $w --no-cpu-baseline --no-e2e --no-digests "$@" > $O/$tag.json 2> $O/$tag.err; python -c "import json;d=json.loads(open('$O/$tag.json').read().strip().splitlines()[-1]);print('$tag',d['value'],d['ms_min'],d['roofline']['frac'],d['verify_mismatched_bytes'],d['tiles'])" 2>&1 | tail -1; }
for rep in 1 2; do
  for w in gpt2-small-tp2-to-pp2 gpt3-1.3b-dp-scaleout; do
    one ${w}_t0_$rep $w RESHARD_TMA_TENSOR=0
    one ${w}_t1_$rep $w RESHARD_TMA_TENSOR=1
  done
done
one cfg3_t0 gpt3-6.7b-tp4pp2-to-tp2pp2dp2 RESHARD_TMA_TENSOR=0 --steps 5 --warmup 3
one cfg3_t1 gpt3-6.7b-tp4pp2-to-tp2pp2dp2 RESHARD_TMA_TENSOR=1 --steps 5 --warmup 3
