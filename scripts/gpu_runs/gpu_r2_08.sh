#!/bin/bash
# round 2, call 8: the driver's default commands (wall-clocked), stress with TP 8
O=gpurun_out/r2_08; mkdir -p $O
s=$(date +%s.%N); timeout 1800 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/ref1.json 2> $O/ref1.err; e=$(date +%s.%N); echo "ref wall $(echo "$e - $s" | bc) s"; tail -c 300 $O/ref1.json
s=$(date +%s.%N); timeout 1800 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $O/n1.json 2> $O/n1.err; e=$(date +%s.%N); echo "ours wall $(echo "$e - $s" | bc) s"; python -c "import json;d=json.load(open('$O/n1.json'));print(d['value'],d['roofline']['frac'],d['e2e']['value'],d['cpu_baseline']['value'],d['host_ms'])"
timeout 1500 python scripts/stress_gpu.py --cases 3000 --seed 2208 > $O/stress.jsonl 2> $O/stress.err; tail -1 $O/stress.jsonl; tail -3 $O/stress.err
