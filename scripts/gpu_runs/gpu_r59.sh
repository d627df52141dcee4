#!/bin/bash
# r59: fabric (NVLink) roofline of the N>1 bench line, ranks sharing one GPU (correctness of
# the accounting; the times themselves are not NVLink times here).
set -u
OUT=gpurun_out/r59
mkdir -p "$OUT"
for n in 2 4; do
  RESHARD_DIST_BACKEND=gloo RESHARD_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n \
    --master-addr 127.0.0.1 --master-port $((29700 + n)) bench.py --gpus $n --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
    > "$OUT/bench_n$n.json" 2> "$OUT/bench_n$n.err"; echo "rc=$?" >> "$OUT/bench_n$n.err"
done
timeout 900 python -m pytest tests/test_gpu_multiprocess.py -m gpu -x -q > "$OUT/pytest_mp.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_mp.log"
echo done > "$OUT/DONE"
