#!/bin/bash
# round 2, call 23: GUIDED dynamic claims (claim = min(8, remaining / (grid * guide))) vs fixed
# 8-tile claims vs the static split, on GPT-2 small, GPT-3 1.3B and the 6.7B recovery; parity
# of the guided kernel (executor suite forced onto bulk_dyn with guide 2)
O=gpurun_out/r2_23; mkdir -p $O
RESHARD_COPY_KERNEL=bulk_dyn RESHARD_DYN_GUIDE=2 python -m pytest tests/test_gpu_executor.py -m gpu -q -x > $O/pytest_guided.txt 2>&1; tail -1 $O/pytest_guided.txt; grep -E "FAILED|rror" $O/pytest_guided.txt | head -5
RESHARD_COPY_KERNEL=bulk_dyn RESHARD_DYN_GUIDE=1 timeout 900 python scripts/stress_gpu.py --cases 800 > $O/stress_guided.txt 2>&1; tail -2 $O/stress_guided.txt
ab() { n=$1; shift; env "$@" timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-digests $W > $O/$n.json 2> $O/ab.err; python -c "import json;d=json.load(open('$O/$n.json'));print('$n',d['value'],d['ms_min'],d['roofline']['frac'],d['roofline']['kernel'],d['verify_mismatched_bytes'])"; }
for r in 1 2; do
for w in gpt2-small-tp2-to-pp2 gpt3-1.3b-dp-scaleout gpt3-6.7b-recovery; do
  W="--workload $w"
  ab ${w}_static_$r RESHARD_DYN_MIN_TILES=0
  ab ${w}_fixed8_$r RESHARD_COPY_KERNEL=bulk_dyn
  for g in 1 2 4; do ab ${w}_guide${g}_$r RESHARD_COPY_KERNEL=bulk_dyn RESHARD_DYN_GUIDE=$g; done
done
done
