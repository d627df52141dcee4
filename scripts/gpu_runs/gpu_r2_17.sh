#!/bin/bash
# round 2, call 17: bulk_dyn tail sweep (static prefix + dynamic tail) vs bulk_strided, same box
O=gpurun_out/r2_17; mkdir -p $O
python -m pytest tests/test_gpu_executor.py -m gpu -q -x -k "bulk_dyn" > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt; grep -E "FAILED|rror" $O/pytest.txt | head -5
ab() { w=$1; k=$2; t=$3; RESHARD_COPY_KERNEL=$k RESHARD_DYN_TAIL=$t timeout 900 python bench.py --workload $w --no-cpu-baseline --no-e2e --no-digests > $O/ab_${w}_${k}_$t.json 2> $O/ab_${w}_${k}_$t.err; python -c "import json;d=json.load(open('$O/ab_${w}_${k}_$t.json'));print('$w $k tail=$t',d['value'],d['ms_min'],d['roofline']['frac'],d['verify_mismatched_bytes'])"; }
for w in gpt2-small-tp2-to-pp2 gpt3-1.3b-dp-scaleout; do
  ab $w bulk_strided 0
  for t in -1 1 2 4 8 16 32; do ab $w bulk_dyn $t; done
  ab $w bulk_strided 0
done
for w in gpt3-6.7b-tp4pp2-to-tp2pp2dp2 gpt3-6.7b-recovery; do
  ab $w bulk_strided 0
  for t in -1 4 16; do ab $w bulk_dyn $t; done
done
