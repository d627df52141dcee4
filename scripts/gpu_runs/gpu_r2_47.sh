#!/bin/bash
# round 2, call 47: 32 KiB stages — ring depth 5 / 6 / 7 on the four copy workloads
O=gpurun_out/r2_47; mkdir -p $O
one() { tag=$1; w=$2; e=$3; shift 3; env $e timeout 900 python bench.py --workload $w --no-cpu-baseline --no-e2e --no-digests "$@" > $O/$tag.json 2> $O/$tag.err; python -c "import json;d=json.loads(open('$O/$tag.json').read().strip().splitlines()[-1]);print('$tag',d['value'],d['ms_min'],d['roofline']['frac'],d['roofline']['kernel'],d['verify_mismatched_bytes'])" 2>&1 | tail -1; }
for rep in 1 2; do for st in 5 6 7; do
  one gpt2_s${st}_$rep gpt2-small-tp2-to-pp2 RESHARD_BULK_STAGES=$st
  one d13_s${st}_$rep gpt3-1.3b-dp-scaleout RESHARD_BULK_STAGES=$st
done; done
for st in 5 6 7; do
  one cfg3_s$st gpt3-6.7b-tp4pp2-to-tp2pp2dp2 RESHARD_BULK_STAGES=$st --steps 5 --warmup 3
  one cfg4_s$st gpt3-6.7b-recovery RESHARD_BULK_STAGES=$st --steps 5 --warmup 3
done
