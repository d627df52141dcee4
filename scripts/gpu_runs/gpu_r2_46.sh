#!/bin/bash
# round 2, call 46: claims of 2 tiles as the default — GPT-2 small static vs dynamic (threshold),
# claim 1 vs 2 on 1.3B, executor tests, compute-sanitizer on the dynamic-claim kernels
O=gpurun_out/r2_46; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_executor.py tests/test_full_size.py -m gpu -q > $O/pytest_exec.txt 2>&1; tail -1 $O/pytest_exec.txt; grep FAILED $O/pytest_exec.txt | head -3
one() { tag=$1; w=$2; e=$3; shift 3; env $e timeout 900 python bench.py --workload $w --no-cpu-baseline --no-e2e --no-digests "$@" > $O/$tag.json 2> $O/$tag.err; python -c "import json;d=json.loads(open('$O/$tag.json').read().strip().splitlines()[-1]);print('$tag',d['value'],d['ms_min'],d['roofline']['frac'],d['roofline']['kernel'],d['verify_mismatched_bytes'])" 2>&1 | tail -1; }
for rep in 1 2; do
  one gpt2_static_$rep gpt2-small-tp2-to-pp2 X=1
  one gpt2_dyn2_$rep gpt2-small-tp2-to-pp2 RESHARD_COPY_KERNEL=bulk_dyn
  one d13_claim1_$rep gpt3-1.3b-dp-scaleout RESHARD_DYN_CLAIM=1
  one d13_claim2_$rep gpt3-1.3b-dp-scaleout X=1
  one d13_claim3_$rep gpt3-1.3b-dp-scaleout RESHARD_DYN_CLAIM=3
done
RESHARD_COPY_KERNEL=bulk_dyn timeout 1200 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_executor.py -m gpu -q -k "random_transitions or fig6" > $O/racecheck_dyn.txt 2>&1; tail -2 $O/racecheck_dyn.txt | head -1
RESHARD_COPY_KERNEL=bulk_dyn timeout 1200 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_executor.py -m gpu -q -k "random_transitions or fig6" > $O/memcheck_dyn.txt 2>&1; tail -2 $O/memcheck_dyn.txt | head -1
