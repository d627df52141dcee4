#!/bin/bash
# r69: K8 at the N/40 window: launch list of one N = 10^8 shuffle and ncu --set full of the
# round-3 reserve and commit launches
set -u
OUT=gpurun_out/r69
mkdir -p "$OUT"
CMD="import paper_2312_05181_b200 as rs; c=rs.Context(1,[0],[0]); p=c.malloc(0,8*10**8); rs.shuffle_epoch_device(c,0,10**8,0x5EED,0,p)"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/k8_launches.csv" python -c "$CMD" > "$OUT/ncu1.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:shuffle_win -s 5 -c 2 -o "$OUT/k8_round3" python -c "$CMD" > "$OUT/ncu2.log" 2>&1
timeout 300 python scripts/probe_k8.py --fracs 40,40 > "$OUT/probe_k8.jsonl" 2> "$OUT/probe_k8.err"
echo done > "$OUT/DONE"
