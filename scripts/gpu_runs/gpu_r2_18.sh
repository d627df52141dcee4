#!/bin/bash
# round 2, call 18: bulk_dyn claim size sweep (all-dynamic) vs bulk_strided, twice each
O=gpurun_out/r2_18; mkdir -p $O
ab() { w=$1; k=$2; b=$3; r=$4; RESHARD_COPY_KERNEL=$k RESHARD_DYN_CLAIM=$b timeout 900 python bench.py --workload $w --no-cpu-baseline --no-e2e --no-digests > $O/ab_${w}_${k}_$b_$r.json 2> $O/ab.err; python -c "import json;d=json.load(open('$O/ab_${w}_${k}_$b_$r.json'));print('$w $k claim=$b',d['value'],d['ms_min'],d['roofline']['frac'],d['verify_mismatched_bytes'])"; }
for r in 1 2; do
for w in gpt2-small-tp2-to-pp2 gpt3-1.3b-dp-scaleout gpt3-6.7b-recovery; do
  ab $w bulk_strided 0 $r
  for b in 1 2 4 8; do ab $w bulk_dyn $b $r; done
done
done
