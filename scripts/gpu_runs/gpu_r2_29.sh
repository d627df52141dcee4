#!/bin/bash
# round 2, call 29: the windowed host-buffer e2e on the GPT-3 6.7B workloads (configs 3 and 4)
O=gpurun_out/r2_29; mkdir -p $O
free -g > $O/free.txt
run() { n=$1; shift; timeout 1500 python bench.py "$@" > $O/$n.json 2> $O/$n.err || echo "$n rc=$?"; python -c "import json;d=json.loads(open('$O/$n.json').read().strip().splitlines()[-1]);e=d.get('e2e') or {};print('$n',d.get('value'),(d.get('roofline') or {}).get('frac'),e.get('value'),(e.get('roofline') or {}).get('frac'),e.get('mismatched_bytes'),e.get('error'),e.get('host_buffers_gb'))" 2>&1 | tail -1; }
run cfg4 --workload gpt3-6.7b-recovery --no-cpu-baseline --steps 5 --warmup 3
run cfg3 --workload gpt3-6.7b-tp4pp2-to-tp2pp2dp2 --no-cpu-baseline --steps 5 --warmup 3
