#!/bin/bash
# round 2, call 31: the skip-unread test after its fix; GPT-2 small host-pipeline trace
O=gpurun_out/r2_31; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_executor.py -m gpu -q -k "run_host" > $O/pytest_run_host.txt 2>&1; tail -2 $O/pytest_run_host.txt
RESHARD_HOST_TRACE=1 timeout 900 python bench.py --workload gpt2-small-tp2-to-pp2 --no-cpu-baseline --e2e-steps 1 > $O/gpt2_trace.json 2> $O/gpt2_trace.err; echo rc=$?
grep -c host-trace $O/gpt2_trace.err
