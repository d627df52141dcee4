#!/bin/bash
# round 2, call 19: the auto switch (bulk_strided -> dynamic claims from 2e5 tiles) and claim 8/16/32
O=gpurun_out/r2_19; mkdir -p $O
python -m pytest tests/test_gpu_executor.py -m gpu -q -x > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt; grep -E "FAILED|rror" $O/pytest.txt | head -5
ab() { n=$1; shift; env "$@" timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-digests $W > $O/$n.json 2> $O/ab.err; python -c "import json;d=json.load(open('$O/$n.json'));print('$n',d['value'],d['ms_min'],d['roofline']['frac'],d['verify_mismatched_bytes'])"; }
for r in 1 2; do
for w in gpt2-small-tp2-to-pp2 gpt3-1.3b-dp-scaleout gpt3-6.7b-tp4pp2-to-tp2pp2dp2 gpt3-6.7b-recovery; do
  W="--workload $w"
  ab ${w}_static_$r RESHARD_DYN_MIN_TILES=0
  ab ${w}_auto_$r RESHARD_DYN_MIN_TILES=200000
  for b in 16 32; do ab ${w}_dyn$b_$r RESHARD_COPY_KERNEL=bulk_dyn RESHARD_DYN_CLAIM=$b; done
done
done
