#!/bin/bash
# round 2, call 6: pipelined run_host_world (parity + emulated A/B), single-process worlds
O=gpurun_out/r2_06; mkdir -p $O
python -m pytest tests/test_gpu_executor.py tests/test_gpu_multiprocess.py -m gpu -q -x > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt; grep -E "FAILED|rror" $O/pytest.txt | head -5
for pl in 1 0; do
  RESHARD_WORLD_PIPELINE=$pl RESHARD_SAME_GPU=1 timeout 900 python bench.py --gpus 4 --no-cpu-baseline --steps 10 > $O/n4_pipe$pl.json 2> $O/n4_pipe$pl.err
  python -c "import json;d=json.load(open('$O/n4_pipe$pl.json'));print('pipe=$pl',d['value'],d['e2e'],d['host_ms'])"; tail -2 $O/n4_pipe$pl.err
done
