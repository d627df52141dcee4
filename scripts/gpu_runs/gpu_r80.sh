#!/bin/bash
# r80: K8 persistent cooperative variant (RESHARD_K8=coop: every round in one launch, grid
# barriers between phases) vs the shipped graph batches
set -u
OUT=gpurun_out/r80
mkdir -p "$OUT"
RESHARD_K8=coop timeout 300 python -m pytest tests/test_dataset.py -m gpu -x -q -k "k8" > "$OUT/pytest_k8_coop.log" 2>&1
RESHARD_K8=coop timeout 600 python scripts/stress_k8.py --cases 500 --seed 80 > "$OUT/stress_k8_coop.jsonl" 2>&1
RESHARD_K8=coop timeout 300 python scripts/probe_k8.py --fracs 80,160,320,640 > "$OUT/probe_k8_coop.jsonl" 2> "$OUT/probe_k8.err"
timeout 300 python scripts/probe_k8.py --fracs 160,320 > "$OUT/probe_k8_graph.jsonl" 2>> "$OUT/probe_k8.err"
RESHARD_K8=coop timeout 300 python scripts/probe_k8.py --n 3000000 --fracs 20,40 > "$OUT/probe_k8_coop_3m.jsonl" 2>> "$OUT/probe_k8.err"
echo done > "$OUT/DONE"
