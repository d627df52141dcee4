#!/bin/bash
# round 2, call 21: dynamic claims in the LDG/STG kernels (K1 aligned / K2 fan-out) — parity and A/B
O=gpurun_out/r2_21; mkdir -p $O
python -m pytest tests/test_gpu_executor.py -m gpu -q -x -k "ldg_dynamic or bulk_dyn or single_process" > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt; grep -E "FAILED|rror" $O/pytest.txt | head -5
ab() { n=$1; shift; env "$@" timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-digests $W > $O/$n.json 2> $O/ab.err; python -c "import json;d=json.load(open('$O/$n.json'));print('$n',d['value'],d['ms_min'],d['roofline']['frac'],d['verify_mismatched_bytes'])"; tail -1 $O/ab.err; }
for r in 1 2; do
  for w in gpt3-1.3b-dp-scaleout gpt3-6.7b-recovery gpt2-small-tp2-to-pp2; do
    W="--workload $w"
    ab ${w}_ldg_static_$r RESHARD_COPY_KERNEL=ldg RESHARD_LDG_DYN=0
    ab ${w}_ldg_dyn_$r RESHARD_COPY_KERNEL=ldg RESHARD_LDG_DYN=1
  done
  W="--gpus 4"
  ab emu4_static_$r RESHARD_SAME_GPU=1 RESHARD_LDG_DYN=0
  ab emu4_dyn_$r RESHARD_SAME_GPU=1 RESHARD_LDG_DYN=1
  W="--gpus 8 --workload gpt3-6.7b-tp4pp2-to-tp2pp2dp2"
  ab emu8_67b_static_$r RESHARD_SAME_GPU=1 RESHARD_LDG_DYN=0
  ab emu8_67b_dyn_$r RESHARD_SAME_GPU=1 RESHARD_LDG_DYN=1
done
