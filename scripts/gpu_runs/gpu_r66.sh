#!/bin/bash
# r66: compute-sanitizer over the final tree: the device-expanded copy schedule (expansion
# kernels), the split K5 (gather pass / ticketed tile scan / blocked finalize), index padding,
# K8, broadcast and central mode.
set -u
OUT=gpurun_out/r66
mkdir -p "$OUT"
S=/usr/local/cuda/bin/compute-sanitizer
run() {  # tool, log name, timeout, pytest args...
  local tool=$1 name=$2 to=$3
  shift 3
  timeout "$to" $S --tool "$tool" --error-exitcode 9 python -m pytest -m gpu -x -q "$@" > "$OUT/${tool}_${name}.log" 2>&1
  echo "rc=$?" >> "$OUT/${tool}_${name}.log"
}
run memcheck executor 2400 tests/test_gpu_executor.py -k "not full_size and not config1 and not 4gib"
run memcheck dataset 1500 tests/test_dataset.py -k "not full_size"
run racecheck executor 1200 tests/test_gpu_executor.py -k "fig6 or single_process or broadcast or central"
run racecheck dataset 1200 tests/test_dataset.py -k "k5_kernel or index_pad or k8"
run synccheck executor 900 tests/test_gpu_executor.py -k "fig6 or single_process or broadcast or central"
run synccheck dataset 900 tests/test_dataset.py -k "k5_kernel or k8"
echo done > "$OUT/DONE"
