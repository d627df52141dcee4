#!/bin/bash
# round 2, call 24: GPT-2 small — is K3d's loss there the single issuing thread meeting runs of
# row-strided tiles (8 consecutive dim-1 TP tiles per claim, 19 bulk copies each way)?  A/B of
# static / dynamic claims with and without K3T tensor-map boxes (one TMA op per box)
O=gpurun_out/r2_24; mkdir -p $O
ab() { n=$1; shift; env "$@" timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-digests $W > $O/$n.json 2> $O/ab.err; python -c "import json;d=json.load(open('$O/$n.json'));print('$n',d['value'],d['ms_min'],d['roofline']['frac'],d['roofline']['kernel'],d['verify_mismatched_bytes'])"; }
for r in 1 2; do
for w in gpt2-small-tp2-to-pp2 gpt3-6.7b-tp4pp2-to-tp2pp2dp2; do
  W="--workload $w"
  ab ${w}_static_$r RESHARD_DYN_MIN_TILES=0
  ab ${w}_static_k3t_$r RESHARD_DYN_MIN_TILES=0 RESHARD_TMA_TENSOR=1
  ab ${w}_warp_$r RESHARD_COPY_KERNEL=bulk_warp
  for c in 2 8; do
    ab ${w}_dyn${c}_$r RESHARD_COPY_KERNEL=bulk_dyn RESHARD_DYN_CLAIM=$c
    ab ${w}_dyn${c}_k3t_$r RESHARD_COPY_KERNEL=bulk_dyn RESHARD_DYN_CLAIM=$c RESHARD_TMA_TENSOR=1
  done
done
done
