#!/bin/bash
# round 2, call 62: arena placement of cells at 256 B (default) / 4 KiB / 32 KiB / 64 KiB
# alignment (tiles start at cell offset + k x 32 KiB), GPT-2 small, 1.3B, recovery; two repetitions
O=gpurun_out/r2_62; mkdir -p $O
one() { tag=$1; w=$2; e=$3; shift 3; env $e timeout 900 python bench.py --workload $w --no-cpu-baseline --no-e2e --no-digests "$@" > $O/$tag.json 2> $O/$tag.err; python -c "import json;d=json.loads(open('$O/$tag.json').read().strip().splitlines()[-1]);print('$tag',d['value'],d['ms_min'],d['roofline']['frac'],d['verify_mismatched_bytes'],d['tiles'])" 2>&1 | tail -1; }
for rep in 1 2; do for a in 256 4096 32768 65536; do
  one gpt2_a${a}_$rep gpt2-small-tp2-to-pp2 RESHARD_CELL_ALIGN=$a
  one d13_a${a}_$rep gpt3-1.3b-dp-scaleout RESHARD_CELL_ALIGN=$a
  one cfg4_a${a}_$rep gpt3-6.7b-recovery RESHARD_CELL_ALIGN=$a --steps 5 --warmup 3
done; done
