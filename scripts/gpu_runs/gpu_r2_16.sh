#!/bin/bash
# round 2, call 16: bulk_dyn (dynamic tile claims) — parity, then same-box A/B vs bulk_strided
O=gpurun_out/r2_16; mkdir -p $O
python -m pytest tests/test_gpu_executor.py -m gpu -q -x -k "bulk_dyn or broadcast" > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt; grep -E "FAILED|rror" $O/pytest.txt | head -5
timeout 900 python scripts/stress_gpu.py --cases 2000 --seed 2216 > $O/stress.jsonl 2> $O/stress.err; tail -1 $O/stress.jsonl; tail -2 $O/stress.err
for rep in 1 2; do
for w in gpt2-small-tp2-to-pp2 gpt3-1.3b-dp-scaleout gpt3-6.7b-tp4pp2-to-tp2pp2dp2 gpt3-6.7b-recovery; do
  for k in bulk_strided bulk_dyn; do
    RESHARD_COPY_KERNEL=$k timeout 900 python bench.py --workload $w --no-cpu-baseline --no-e2e --no-digests > $O/ab_${w}_${k}_$rep.json 2> $O/ab_${w}_${k}_$rep.err
    python -c "import json;d=json.load(open('$O/ab_${w}_${k}_$rep.json'));print('$w $k',d['value'],d['ms_min'],d['roofline']['frac'],d['verify_mismatched_bytes'])"
  done
done
done
