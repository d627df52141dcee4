#!/bin/bash
# r33: dataset bench through torchrun with 2 ranks sharing one GPU (gloo) + default bench line.
set -u
TAG=${1:-r33}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
RESHARD_DIST_BACKEND=gloo RESHARD_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 \
  --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline \
  --workload dataset-100m-dp2to4to8 > "$OUT/bench_dataset_n2.json" 2> "$OUT/bench_dataset_n2.err"; echo "rc=$?" >> "$OUT/bench_dataset_n2.err"
timeout 600 python bench.py --no-cpu-baseline > "$OUT/bench.json" 2> "$OUT/bench.err"
echo done > "$OUT/DONE"
