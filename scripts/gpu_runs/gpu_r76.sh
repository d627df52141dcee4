#!/bin/bash
# r76: K8 commit kernel unrolled by two (both loads before either check)
set -u
OUT=gpurun_out/r76
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_dataset.py -m gpu -x -q > "$OUT/pytest_dataset.log" 2>&1
timeout 900 python scripts/stress_k8.py --cases 1000 --seed 74 > "$OUT/stress_k8.jsonl" 2>&1
timeout 600 python scripts/probe_k8.py --fracs 80,160,320,640 > "$OUT/probe_k8.jsonl" 2> "$OUT/probe_k8.err"
timeout 600 python scripts/probe_k8.py --n 3000000 --fracs 20,40 > "$OUT/probe_k8_3m.jsonl" 2>> "$OUT/probe_k8.err"
CMD="import paper_2312_05181_b200 as rs; c=rs.Context(1,[0],[0]); p=c.malloc(0,8*10**8); rs.shuffle_epoch_device(c,0,10**8,0x5EED,0,p)"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file "$OUT/k8_launches.csv" python -c "$CMD" > "$OUT/ncu1.log" 2>&1
echo done > "$OUT/DONE"
