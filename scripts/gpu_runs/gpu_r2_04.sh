#!/bin/bash
# round 2, call 4: the whole GPU suite + smoke, host-work trace of the default workload, the 6.7B
# recovery reference arm (failed devices unfilled), the default workload's launch list
O=gpurun_out/r2_04; mkdir -p $O
python -m pytest tests -m gpu -q > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt; grep -E "FAILED|Error" $O/pytest.txt | head
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -2 $O/smoke.txt
RESHARD_HOST_TRACE=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 > $O/bench_trace.json 2> $O/bench_trace.err; grep -E "lower-trace|prepare-trace" $O/bench_trace.err | head; python -c "import json;d=json.load(open('$O/bench_trace.json'));print(d['value'],d['host_ms'])"
timeout 1500 python bench.py --impl reference --workload gpt3-6.7b-recovery --steps 2 --warmup 3 > $O/ref_recovery.json 2> $O/ref_recovery.err; tail -c 700 $O/ref_recovery.json; tail -2 $O/ref_recovery.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/launches.out 2>&1; tail -1 $O/launches.out | cut -c1-300
