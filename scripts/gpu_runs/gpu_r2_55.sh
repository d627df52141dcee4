#!/bin/bash
# round 2, call 55: GPT-2 small e2e vs host chunk count (24 / 32 / 64), three repetitions each,
# interleaved; e2e-steps 5
O=gpurun_out/r2_55; mkdir -p $O
for rep in 1 2 3; do for c in 24 32 64; do
  RESHARD_HOST_CHUNKS=$c timeout 600 python bench.py --workload gpt2-small-tp2-to-pp2 --no-cpu-baseline --no-digests --e2e-steps 5 > $O/gpt2_c${c}_$rep.json 2> $O/gpt2_c${c}_$rep.err
  python -c "import json;d=json.loads(open('$O/gpt2_c${c}_$rep.json').read().strip().splitlines()[-1]);e=d['e2e'];print('chunks=$c rep=$rep',e['value'],e['roofline'].get('bidir_gbs_each'),e['roofline'].get('frac'))"
done; done
