#!/bin/bash
# round 2, call 11: torchrun world timing through interprocess events (2 and 4 ranks sharing cuda:0)
O=gpurun_out/r2_11; mkdir -p $O
python -m pytest tests/test_gpu_multiprocess.py -m gpu -q -x -k ipc_push > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt; grep -E "FAILED|rror" $O/pytest.txt | head -5
for n in 2 4; do
  RESHARD_SAME_GPU=1 RESHARD_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 29$n$n$n bench.py --gpus $n --steps 5 --no-cpu-baseline > $O/tr_$n.json 2> $O/tr_$n.err
  python -c "import json;d=json.loads(open('$O/tr_$n.json').read().strip().splitlines()[-1]);print($n,d['value'],d['ms_max_gpu_kernel'],d['timing'][:40],d['e2e'].get('value'),d['e2e'].get('path','')[:60])"; tail -2 $O/tr_$n.err
done
