#!/bin/bash
# r48: leaner host lowering / descriptor upload — executor + multiprocess suites, host_ms.
set -u
OUT=gpurun_out/r48
mkdir -p "$OUT"
timeout 1200 python -m pytest tests/test_gpu_executor.py tests/test_gpu_multiprocess.py tests/test_central_mode.py -m gpu -x -q > "$OUT/pytest.log" 2>&1; echo "rc=$?" >> "$OUT/pytest.log"
timeout 600 python bench.py --no-cpu-baseline > "$OUT/bench.json" 2> "$OUT/bench.err"
timeout 900 python bench.py --workload gpt3-6.7b-tp4pp2-to-tp2pp2dp2 --no-cpu-baseline > "$OUT/bench_67b.json" 2>> "$OUT/bench.err"
timeout 600 python bench.py --workload gpt2-small-tp2-to-pp2 --no-cpu-baseline > "$OUT/bench_gpt2.json" 2>> "$OUT/bench.err"
timeout 900 python scripts/stress_gpu.py --cases 3000 --seed 11 > "$OUT/stress.jsonl" 2>&1
echo done > "$OUT/DONE"
