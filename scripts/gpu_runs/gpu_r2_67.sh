#!/bin/bash
# round 2, call 67: the final tree — GPU suite (incl. acceptance #10), smoke, default line
O=gpurun_out/r2_67; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest.txt 2>&1; tail -1 $O/pytest.txt; grep FAILED $O/pytest.txt | head
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -2 $O/smoke.txt
timeout 1200 python bench.py > $O/default.json 2> $O/default.err; python -c "import json;d=json.loads(open('$O/default.json').read().strip().splitlines()[-1]);print(d['value'],d['roofline']['frac'],d['e2e']['value'],d['e2e']['roofline']['frac'],d['cpu_baseline']['value'],d['verify_mismatched_bytes'],d['execution_report']['match'],d['clocks'])"
