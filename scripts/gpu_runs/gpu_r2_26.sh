#!/bin/bash
# round 2, call 26: static split with runs of K consecutive tiles per CTA (runs c, c+grid, ...):
# dynamic claims' per-CTA locality without the counter; K = 1 (shipped), 2, 4, 8, 16 vs K3d
O=gpurun_out/r2_26; mkdir -p $O
RESHARD_DYN_MIN_TILES=0 RESHARD_RUN_SHIFT=3 python -m pytest tests/test_gpu_executor.py tests/test_full_size.py -m gpu -q -x > $O/pytest_run8.txt 2>&1; tail -1 $O/pytest_run8.txt; grep -E "FAILED|rror" $O/pytest_run8.txt | head -5
RESHARD_RUN_SHIFT=2 timeout 900 python scripts/stress_gpu.py --cases 800 > $O/stress_run4.txt 2>&1; tail -1 $O/stress_run4.txt
ab() { n=$1; shift; env "$@" timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-digests $W > $O/$n.json 2> $O/ab.err; python -c "import json;d=json.load(open('$O/$n.json'));print('$n',d['value'],d['ms_min'],d['roofline']['frac'],d['verify_mismatched_bytes'])"; }
for r in 1 2; do
for w in gpt2-small-tp2-to-pp2 gpt3-1.3b-dp-scaleout gpt3-6.7b-recovery gpt3-6.7b-tp4pp2-to-tp2pp2dp2; do
  W="--workload $w"
  ab ${w}_dyn8_$r RESHARD_COPY_KERNEL=bulk_dyn
  for k in 0 1 2 3 4; do ab ${w}_run${k}_$r RESHARD_DYN_MIN_TILES=0 RESHARD_RUN_SHIFT=$k; done
done
done
