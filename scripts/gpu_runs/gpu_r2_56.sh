#!/bin/bash
# round 2, call 56: minimum host chunk of 44 MiB — run_host GPU tests, GPT-2 small and 1.3B e2e
O=gpurun_out/r2_56; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_executor.py -m gpu -q -k "run_host" > $O/pytest_run_host.txt 2>&1; tail -1 $O/pytest_run_host.txt
for rep in 1 2 3; do
  timeout 600 python bench.py --workload gpt2-small-tp2-to-pp2 --no-cpu-baseline --no-digests --e2e-steps 5 > $O/gpt2_$rep.json 2> $O/gpt2_$rep.err
  python -c "import json;d=json.loads(open('$O/gpt2_$rep.json').read().strip().splitlines()[-1]);e=d['e2e'];print('gpt2 rep=$rep',e['value'],e['roofline'].get('frac'),e['mismatched_bytes'])"
done
timeout 900 python bench.py --no-cpu-baseline --no-digests > $O/default.json 2> $O/default.err
python -c "import json;d=json.loads(open('$O/default.json').read().strip().splitlines()[-1]);e=d['e2e'];print('default',d['value'],e['value'],e['roofline'].get('frac'),e['mismatched_bytes'])"
