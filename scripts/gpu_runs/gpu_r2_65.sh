#!/bin/bash
# round 2, call 65: the driver's multi-GPU commands on a one-GPU box run emulated and labelled
# (no RESHARD_SAME_GPU in the environment): plain --gpus 2, torchrun 2 ranks, the dataset workload
O=gpurun_out/r2_65; mkdir -p $O
unset RESHARD_SAME_GPU
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > $O/plain_n2.json 2> $O/plain_n2.err; echo plain rc=$?
python -c "import json;d=json.loads(open('$O/plain_n2.json').read().strip().splitlines()[-1]);print(d['n_gpus'],d['value'],d['emulated_on_one_gpu'],d['emulation'],d['verify_mismatched_bytes'])"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > $O/torchrun_n2.json 2> $O/torchrun_n2.err; echo torchrun rc=$?
python -c "import json;d=json.loads([l for l in open('$O/torchrun_n2.json').read().splitlines() if l.startswith('{')][-1]);print(d['n_gpus'],d['value'],d['emulated_on_one_gpu'],d['emulation'],d['verify_mismatched_bytes'],d['timing'][:40])"
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --workload dataset-100m-dp2to4to8 --no-cpu-baseline --no-e2e > $O/dataset_n2.json 2> $O/dataset_n2.err; echo dataset rc=$?
python -c "import json;d=json.loads([l for l in open('$O/dataset_n2.json').read().splitlines() if l.startswith('{')][-1]);print(d['n_gpus'],d['value'],d['emulation'],d['spot_check'])"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29612 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > $O/ref_n2.json 2> $O/ref_n2.err; echo ref rc=$?; tail -c 300 $O/ref_n2.json
