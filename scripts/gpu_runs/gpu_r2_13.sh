#!/bin/bash
# round 2, call 13: shift-ordered peer lists — parity (executor suite, multiprocess, stress)
O=gpurun_out/r2_13; mkdir -p $O
python -m pytest tests/test_gpu_executor.py tests/test_gpu_multiprocess.py -m gpu -q -x > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt; grep -E "FAILED|rror" $O/pytest.txt | head -5
timeout 1500 python scripts/stress_gpu.py --cases 5000 --seed 2213 > $O/stress.jsonl 2> $O/stress.err; tail -1 $O/stress.jsonl; tail -3 $O/stress.err
RESHARD_SAME_GPU=1 timeout 900 python bench.py --gpus 8 --workload gpt3-6.7b-tp4pp2-to-tp2pp2dp2 --no-cpu-baseline --steps 5 > $O/n8_67b.json 2> $O/n8_67b.err; python -c "import json;d=json.load(open('$O/n8_67b.json'));print(d['value'],d['waves'],d['verify_mismatched_bytes'],d['fabric']['t_roof_ms'],d['roofline']['frac'],d['host_ms'])"; tail -2 $O/n8_67b.err
