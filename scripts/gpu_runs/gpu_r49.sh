#!/bin/bash
# r49: device-resident copy schedule (pieces expanded into tiles on the GPU) — GPU suite,
# stress, benches with host times.
set -u
OUT=gpurun_out/r49
mkdir -p "$OUT"
timeout 1800 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_gpu.log"
timeout 900 python scripts/stress_gpu.py --cases 6000 --seed 31 > "$OUT/stress.jsonl" 2>&1
RESHARD_HOST_TRACE=1 timeout 600 python bench.py --no-cpu-baseline > "$OUT/bench.json" 2> "$OUT/trace.err"
timeout 900 python bench.py --workload gpt3-6.7b-tp4pp2-to-tp2pp2dp2 --no-cpu-baseline > "$OUT/bench_67b.json" 2>> "$OUT/bench.err"
timeout 600 python bench.py --workload gpt2-small-tp2-to-pp2 --no-cpu-baseline > "$OUT/bench_gpt2.json" 2>> "$OUT/bench.err"
timeout 600 python bench.py --workload gpt3-1.3b-dp-scaleout --mode central --no-cpu-baseline > "$OUT/bench_central.json" 2>> "$OUT/bench.err"
timeout 600 env RESHARD_COPY_KERNEL=bulk python bench.py --no-cpu-baseline > "$OUT/bench_bulkvariant.json" 2>> "$OUT/bench.err"
echo done > "$OUT/DONE"
