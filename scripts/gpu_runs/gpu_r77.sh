#!/bin/bash
# r77: ncu --set full of the shipped K8 (round-3 reserve and commit launches, N = 10^8)
set -u
OUT=gpurun_out/r77
mkdir -p "$OUT"
CMD="import paper_2312_05181_b200 as rs; c=rs.Context(1,[0],[0]); p=c.malloc(0,8*10**8); rs.shuffle_epoch_device(c,0,10**8,0x5EED,0,p)"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:shuffle_win -s 5 -c 2 -o "$OUT/k8_round3" python -c "$CMD" > "$OUT/ncu.log" 2>&1
echo done > "$OUT/DONE"
