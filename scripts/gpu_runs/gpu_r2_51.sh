#!/bin/bash
# round 2, call 51: the final copy defaults (6 x 32 KiB stages, claims of 2) under the data-plane
# stress (random transitions, every copy kernel, 1-8 GPU worlds, digests) and compute-sanitizer
O=gpurun_out/r2_51; mkdir -p $O
timeout 3000 python scripts/stress_gpu.py --cases 10000 --seed 2051 > $O/stress_gpu.jsonl 2> $O/stress_gpu.err; tail -1 $O/stress_gpu.jsonl; tail -2 $O/stress_gpu.err
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 10 python -m pytest tests/test_gpu_executor.py -m gpu -q -k "random_transitions or fig6 or broadcast or run_host" > $O/${tool}_executor.txt 2>&1; grep -h SUMMARY $O/${tool}_executor.txt | head -1
done
