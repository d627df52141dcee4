#!/bin/bash
# r22: the N>1 bench path at N = 4 and 8 ranks sharing cuda:0 (gloo plumbing, IPC pushes):
# correctness of the torchrun code path for the driver's scaling run, default workload + 6.7B.
set -u
TAG=${1:-r22}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
for n in 4 8; do
  RESHARD_DIST_BACKEND=gloo RESHARD_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n \
    --master-addr 127.0.0.1 --master-port $((29500 + n)) bench.py --gpus $n --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
    > "$OUT/bench_n$n.json" 2> "$OUT/bench_n$n.err"; echo "rc=$?" >> "$OUT/bench_n$n.err"
done
RESHARD_DIST_BACKEND=gloo RESHARD_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=8 \
    --master-addr 127.0.0.1 --master-port 29600 bench.py --gpus 8 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
    --workload gpt3-6.7b-tp4pp2-to-tp2pp2dp2 > "$OUT/bench_67b_n8.json" 2> "$OUT/bench_67b_n8.err"; echo "rc=$?" >> "$OUT/bench_67b_n8.err"
echo done > "$OUT/DONE"
