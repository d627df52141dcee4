#!/bin/bash
# r68: windowed K8 as the only variant (window N/100, scratch N + 2 x N/20 entries): tests,
# dataset stress (K8 on random (n, seed, epoch) every 10th case), window sweep, dataset bench
set -u
OUT=gpurun_out/r68
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_dataset.py -m gpu -x -q > "$OUT/pytest_dataset.log" 2>&1
timeout 900 python scripts/stress_dataset.py --cases 400 --seed 68 > "$OUT/stress_dataset.jsonl" 2> "$OUT/stress_dataset.err"
timeout 600 python scripts/probe_k8.py > "$OUT/probe_k8.jsonl" 2> "$OUT/probe_k8.err"
timeout 600 python bench.py --workload dataset-100m-dp2to4to8 > "$OUT/bench_dataset.json" 2> "$OUT/bench_dataset.err"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "rc=$?" >> "$OUT/smoke.log"
echo done > "$OUT/DONE"
