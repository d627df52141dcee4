#!/bin/bash
# round 2, call 53: long stress runs on the final tree — data plane (40,000 random transitions)
# and dataset (6,000 random cases incl. multi-rank batches)
O=gpurun_out/r2_53; mkdir -p $O
timeout 3000 python scripts/stress_gpu.py --cases 40000 --seed 2053 > $O/stress_gpu.jsonl 2> $O/stress_gpu.err; tail -1 $O/stress_gpu.jsonl; tail -2 $O/stress_gpu.err
timeout 2400 python scripts/stress_dataset.py --cases 6000 --seed 2053 > $O/stress_dataset.jsonl 2> $O/stress_dataset.err; tail -1 $O/stress_dataset.jsonl; tail -2 $O/stress_dataset.err
