#!/bin/bash
# round 2, call 27: compute-sanitizer memcheck / racecheck / synccheck of K3d (dynamic tile
# claims, the default for launches of >= 2e5 tiles) — the executor suite forced onto bulk_dyn
# (small launches, so every claim path incl. the counter reset runs), plus the LDG/STG kernels
# with dynamic claims
O=gpurun_out/r2_27; mkdir -p $O
for tool in memcheck racecheck synccheck; do
  RESHARD_COPY_KERNEL=bulk_dyn RESHARD_LDG_DYN=1 timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest tests/test_gpu_executor.py -m gpu -q -k "not larger_than_4gib and not full_size" > $O/sanitizer_$tool.txt 2>&1; echo "$tool rc=$?"; tail -2 $O/sanitizer_$tool.txt
done
