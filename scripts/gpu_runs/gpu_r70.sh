#!/bin/bash
# r70: K8 with packed reservations (high word of the permutation entry) vs separate
# reservations (RESHARD_K8=sep, retired after this run): tests, window sweeps, launch list
set -u
OUT=gpurun_out/r70
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_dataset.py -m gpu -x -q -k "k8 or config5" > "$OUT/pytest_k8.log" 2>&1
RESHARD_K8=sep timeout 600 python -m pytest tests/test_dataset.py -m gpu -x -q -k "k8" > "$OUT/pytest_k8_sep.log" 2>&1
timeout 600 python scripts/probe_k8.py --fracs 10,20,40,80,160 > "$OUT/probe_k8_packed.jsonl" 2> "$OUT/probe_k8.err"
RESHARD_K8=sep timeout 600 python scripts/probe_k8.py --fracs 40,40 > "$OUT/probe_k8_sep.jsonl" 2>> "$OUT/probe_k8.err"
timeout 600 python scripts/probe_k8.py --n 3000000 --fracs 10,20,40,80 > "$OUT/probe_k8_3m.jsonl" 2>> "$OUT/probe_k8.err"
CMD="import paper_2312_05181_b200 as rs; c=rs.Context(1,[0],[0]); p=c.malloc(0,8*10**8); rs.shuffle_epoch_device(c,0,10**8,0x5EED,0,p)"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file "$OUT/k8_launches.csv" python -c "$CMD" > "$OUT/ncu1.log" 2>&1
echo done > "$OUT/DONE"
