#!/bin/bash
# r12: full GPU suite after the API-completeness work, default bench + reference arm, and the
# random-gather probe that bounds K5.  Usage: gpurun -- 'bash scripts/gpu_runs/gpu_r12.sh'
set -u
TAG=${1:-r12}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 1500 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python __graft_entry__.py --smoke > "$OUT/smoke.log" 2>&1; echo "rc=$?" >> "$OUT/smoke.log"
timeout 600 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
timeout 600 python bench.py --impl reference > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
timeout 300 scripts/probe_gather > "$OUT/probe_gather.jsonl" 2>&1
timeout 300 scripts/probe_gather 4500000 >> "$OUT/probe_gather.jsonl" 2>&1
echo done > "$OUT/DONE"
