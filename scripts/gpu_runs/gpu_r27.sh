#!/bin/bash
# r27: K8 shuffle per-round launch list (N = 10^8).
set -u
export PYTHONPATH=$PWD
TAG=${1:-r27}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
cat > "$OUT/k8.py" <<'PY'
import paper_2312_05181_b200 as rs
ctx = rs.Context(1, [0], [0])
n = 100_000_000
p = ctx.malloc(0, 8 * n)
for _ in range(2):
    t = rs.shuffle_epoch_device(ctx, 0, n, 0x5EED, 0, p)
print(t)
PY
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none -k regex:shuffle \
  --csv --log-file "$OUT/k8_launches.csv" python "$OUT/k8.py" > "$OUT/k8.log" 2>&1
timeout 300 python "$OUT/k8.py" > "$OUT/k8_plain.log" 2>&1
echo done > "$OUT/DONE"
