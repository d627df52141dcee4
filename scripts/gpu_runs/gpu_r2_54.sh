#!/bin/bash
# round 2, call 54: PCIe rates by transfer size (is the host pipeline's steady rate with 23 MB
# chunks the link's small-transfer rate?), and the GPT-2 small e2e at 16 / 32 / 64 chunks
O=gpurun_out/r2_54; mkdir -p $O
timeout 600 python scripts/probe_pcie_sizes.py > $O/pcie_sizes.jsonl 2> $O/pcie_sizes.err; cat $O/pcie_sizes.jsonl
for c in 16 32 64 128; do
  RESHARD_HOST_CHUNKS=$c timeout 600 python bench.py --workload gpt2-small-tp2-to-pp2 --no-cpu-baseline --no-digests > $O/gpt2_c$c.json 2> $O/gpt2_c$c.err
  python -c "import json;d=json.loads(open('$O/gpt2_c$c.json').read().strip().splitlines()[-1]);e=d['e2e'];print('chunks=$c',e['value'],e['roofline'].get('bidir_gbs_each'),e['roofline'].get('frac'))"
done
