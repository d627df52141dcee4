#!/bin/bash
# round 2, call 12: digests from either DP copy, bench execution_report, a long stress
O=gpurun_out/r2_12; mkdir -p $O
python -m pytest tests/test_gpu_executor.py -m gpu -q -x -k "digests or run_host_world" > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt
timeout 900 python bench.py --no-cpu-baseline > $O/n1.json 2> $O/n1.err; python -c "import json;d=json.load(open('$O/n1.json'));print(d['value'],d['execution_report'],d['e2e']['value'])"; tail -2 $O/n1.err
timeout 2400 python scripts/stress_gpu.py --cases 20000 --seed 2212 > $O/stress.jsonl 2> $O/stress.err; tail -1 $O/stress.jsonl; tail -3 $O/stress.err
