#!/bin/bash
# round 2, call 7: torchrun paths with the world-API e2e, config 1 both arms, the driver's own
# default commands (timed)
O=gpurun_out/r2_07; mkdir -p $O
python -m pytest tests/test_gpu_multiprocess.py -m gpu -q -x > $O/pytest_mp.txt 2>&1; tail -2 $O/pytest_mp.txt; grep -E "FAILED|rror" $O/pytest_mp.txt | head -5
timeout 900 python bench.py --workload gpt2-small-tp2-to-pp2 > $O/gpt2.json 2> $O/gpt2.err; tail -c 1200 $O/gpt2.json
timeout 900 python bench.py --impl reference --workload gpt2-small-tp2-to-pp2 > $O/gpt2_ref.json 2> $O/gpt2_ref.err; tail -c 400 $O/gpt2_ref.json
/usr/bin/time -f "ref wall %e s" timeout 1800 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/ref1.json 2> $O/ref1.err; tail -1 $O/ref1.err; tail -c 300 $O/ref1.json
/usr/bin/time -f "ours wall %e s" timeout 1800 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $O/n1.json 2> $O/n1.err; tail -1 $O/n1.err; python -c "import json;d=json.load(open('$O/n1.json'));print(d['value'],d['roofline']['frac'],d['e2e']['value'],d['cpu_baseline']['value'],d['host_ms'])"
