#!/bin/bash
# round 2, call 1: the new multi-GPU bench paths + parity suite on one B200
O=gpurun_out/r2_01; mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt
timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err; tail -c 3000 $O/bench_n1.json
RESHARD_SAME_GPU=1 timeout 900 python bench.py --gpus 4 --no-cpu-baseline > $O/bench_n4_same.json 2> $O/bench_n4_same.err; tail -c 2500 $O/bench_n4_same.json; tail -5 $O/bench_n4_same.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; tail -c 1500 $O/bench_ref.json; tail -3 $O/bench_ref.err
