#!/bin/bash
# round 2, call 5: stress of the new paths (K2 fan-out, K3T, DP 8, digests) + compute-sanitizer
# memcheck / racecheck of the new kernels
O=gpurun_out/r2_05; mkdir -p $O
timeout 1500 python scripts/stress_gpu.py --cases 3000 --seed 2202 > $O/stress.jsonl 2> $O/stress.err; tail -2 $O/stress.jsonl; tail -3 $O/stress.err
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest tests/test_gpu_executor.py -m gpu -q -k "tma_tensor or digests or single_process_multi_gpu or broadcast or fig6" > $O/sanitizer_$tool.txt 2>&1; echo "$tool rc=$?"; tail -3 $O/sanitizer_$tool.txt
done
