#!/bin/bash
# round 2, call 30: RS_HOST_SKIP_UNREAD (upload only the source ranges the tiles read) — executor
# GPU tests, then the e2e of the default, GPT-2 small and the recovery workloads
O=gpurun_out/r2_30; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_executor.py -m gpu -q > $O/pytest_executor.txt 2>&1; tail -2 $O/pytest_executor.txt; grep FAILED $O/pytest_executor.txt | head
run() { n=$1; shift; timeout 1500 python bench.py "$@" > $O/$n.json 2> $O/$n.err || echo "$n rc=$?"; python -c "import json;d=json.loads(open('$O/$n.json').read().strip().splitlines()[-1]);e=d.get('e2e') or {};print('$n',d.get('value'),(d.get('roofline') or {}).get('frac'),e.get('value'),(e.get('roofline') or {}).get('frac'),e.get('h2d_bytes_per_step'),e.get('d2h_bytes_per_step'),e.get('ms_full_src_upload'),e.get('mismatched_bytes'),e.get('error'))" 2>&1 | tail -1; }
run cfg4 --workload gpt3-6.7b-recovery --no-cpu-baseline --steps 5 --warmup 3
run default --no-cpu-baseline
run gpt2 --workload gpt2-small-tp2-to-pp2 --no-cpu-baseline
