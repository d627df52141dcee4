#!/bin/bash
# round 2, call 57: same-box A/B of the minimum host chunk (44 MiB vs none) on the GPT-2 small
# and the default e2e, interleaved, three repetitions
O=gpurun_out/r2_57; mkdir -p $O
for rep in 1 2 3; do for m in 44 0; do
  RESHARD_HOST_MIN_CHUNK_MIB=$m timeout 600 python bench.py --workload gpt2-small-tp2-to-pp2 --no-cpu-baseline --no-digests --e2e-steps 5 > $O/gpt2_m${m}_$rep.json 2> $O/gpt2_m${m}_$rep.err
  python -c "import json;d=json.loads(open('$O/gpt2_m${m}_$rep.json').read().strip().splitlines()[-1]);e=d['e2e'];print('gpt2 min=$m rep=$rep',e['value'],e['roofline'].get('frac'))"
done; done
for rep in 1 2; do for m in 44 0; do
  RESHARD_HOST_MIN_CHUNK_MIB=$m timeout 900 python bench.py --no-cpu-baseline --no-digests --e2e-steps 3 > $O/d13_m${m}_$rep.json 2> $O/d13_m${m}_$rep.err
  python -c "import json;d=json.loads(open('$O/d13_m${m}_$rep.json').read().strip().splitlines()[-1]);e=d['e2e'];print('1.3B min=$m rep=$rep',e['value'],e['roofline'].get('frac'))"
done; done
