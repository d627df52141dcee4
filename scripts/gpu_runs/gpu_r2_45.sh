#!/bin/bash
# round 2, call 45: K3d claim size at 32 KiB tiles on the 6.7B workloads and 1.3B (claims of
# 2 / 4 / 8 tiles), and the static split on 6.7B
O=gpurun_out/r2_45; mkdir -p $O
one() { tag=$1; w=$2; e=$3; shift 3; env $e timeout 900 python bench.py --workload $w --no-cpu-baseline --no-e2e --no-digests "$@" > $O/$tag.json 2> $O/$tag.err; python -c "import json;d=json.loads(open('$O/$tag.json').read().strip().splitlines()[-1]);print('$tag',d['value'],d['ms_min'],d['roofline']['frac'],d['roofline']['kernel'],d['verify_mismatched_bytes'])" 2>&1 | tail -1; }
for c in 2 4 8; do
  one cfg3_claim$c gpt3-6.7b-tp4pp2-to-tp2pp2dp2 RESHARD_DYN_CLAIM=$c --steps 5 --warmup 3
  one cfg4_claim$c gpt3-6.7b-recovery RESHARD_DYN_CLAIM=$c --steps 5 --warmup 3
  one d13_claim$c gpt3-1.3b-dp-scaleout RESHARD_DYN_CLAIM=$c
done
one cfg3_static gpt3-6.7b-tp4pp2-to-tp2pp2dp2 RESHARD_DYN_MIN_TILES=0 --steps 5 --warmup 3
one cfg4_static gpt3-6.7b-recovery RESHARD_DYN_MIN_TILES=0 --steps 5 --warmup 3
for c in 2 4 8; do one d13_claim${c}_b gpt3-1.3b-dp-scaleout RESHARD_DYN_CLAIM=$c; done
