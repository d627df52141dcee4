#!/bin/bash
# round 2, call 44: the 6 x 32 KiB default — executor / full-size / multiprocess GPU tests; the
# dynamic-claim size and threshold re-checked at the new tile size; ncu of the default launch
O=gpurun_out/r2_44; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest.txt 2>&1; tail -1 $O/pytest.txt; grep FAILED $O/pytest.txt | head -3
one() { tag=$1; w=$2; shift 2; env "$@" timeout 900 python bench.py --workload $w --no-cpu-baseline --no-e2e --no-digests > $O/$tag.json 2> $O/$tag.err; python -c "import json;d=json.loads(open('$O/$tag.json').read().strip().splitlines()[-1]);print('$tag',d['value'],d['ms_min'],d['roofline']['frac'],d['roofline']['kernel'],d['verify_mismatched_bytes'])" 2>&1 | tail -1; }
for rep in 1 2; do
  one d13_dyn8_$rep gpt3-1.3b-dp-scaleout X=1
  one d13_dyn4_$rep gpt3-1.3b-dp-scaleout RESHARD_DYN_CLAIM=4
  one d13_dyn16_$rep gpt3-1.3b-dp-scaleout RESHARD_DYN_CLAIM=16
  one d13_static_$rep gpt3-1.3b-dp-scaleout RESHARD_DYN_MIN_TILES=0
  one gpt2_static_$rep gpt2-small-tp2-to-pp2 X=1
  one gpt2_dyn8_$rep gpt2-small-tp2-to-pp2 RESHARD_COPY_KERNEL=bulk_dyn
done
one cfg3_dyn8 gpt3-6.7b-tp4pp2-to-tp2pp2dp2 X=1 --steps 5 --warmup 3
one cfg3_static gpt3-6.7b-tp4pp2-to-tp2pp2dp2 RESHARD_DYN_MIN_TILES=0 --steps 5 --warmup 3
timeout 900 ncu --kernel-name regex:"copy_bulk" --launch-skip 3 --launch-count 1 --set full --clock-control none --import-source on \
  -o $O/copy_default python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-digests > $O/copy_ncu.out 2>&1; echo ncu rc=$?
