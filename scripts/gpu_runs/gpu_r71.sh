#!/bin/bash
# r71: K8 packed reservations only, rounds replayed as 6-round graphs with the state check one
# batch behind: tests, dataset stress, window sweeps, L2 fetch-granularity A/B, launch list
set -u
OUT=gpurun_out/r71
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_dataset.py -m gpu -x -q -k "k8 or config5" > "$OUT/pytest_k8.log" 2>&1
timeout 900 python scripts/stress_dataset.py --cases 300 --seed 71 > "$OUT/stress_dataset.jsonl" 2> "$OUT/stress_dataset.err"
timeout 600 python scripts/probe_k8.py --fracs 40,80,160,320,640 > "$OUT/probe_k8.jsonl" 2> "$OUT/probe_k8.err"
RESHARD_L2_FETCH=32 timeout 600 python scripts/probe_k8.py --fracs 160,320 > "$OUT/probe_k8_l2f32.jsonl" 2>> "$OUT/probe_k8.err"
timeout 600 python scripts/probe_k8.py --n 3000000 --fracs 20,40,80,160 > "$OUT/probe_k8_3m.jsonl" 2>> "$OUT/probe_k8.err"
timeout 600 python scripts/probe_k8.py --n 100000 --fracs 1,2,4 > "$OUT/probe_k8_100k.jsonl" 2>> "$OUT/probe_k8.err"
CMD="import paper_2312_05181_b200 as rs; c=rs.Context(1,[0],[0]); p=c.malloc(0,8*10**8); rs.shuffle_epoch_device(c,0,10**8,0x5EED,0,p)"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file "$OUT/k8_launches.csv" python -c "$CMD" > "$OUT/ncu1.log" 2>&1
echo done > "$OUT/DONE"
