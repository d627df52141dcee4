#!/bin/bash
# round 2, call 41: consolidated evidence on the final tree — GPU suite, smoke, every workload's
# line (both arms), emulated 2/4/8-GPU worlds, the default workload's launch list, ncu of the
# fused K5 gather pass, a dataset stress run incl. the multi-rank batches
O=gpurun_out/r2_48; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt; grep -E "FAILED" $O/pytest.txt | head
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -2 $O/smoke.txt
run() { n=$1; shift; timeout 2400 python bench.py "$@" > $O/$n.json 2> $O/$n.err || echo "$n rc=$?"; python -c "import json;d=json.loads(open('$O/$n.json').read().strip().splitlines()[-1]);e=d.get('e2e') or {};print('$n',d.get('value'),(d.get('roofline') or {}).get('frac'),e.get('value'),(e.get('roofline') or {}).get('frac'),(d.get('cpu_baseline') or {}).get('value'))" 2>&1 | tail -1; }
run ref_default --impl reference
run default
run gpt2 --workload gpt2-small-tp2-to-pp2
run ref_gpt2 --impl reference --workload gpt2-small-tp2-to-pp2
run cfg3 --workload gpt3-6.7b-tp4pp2-to-tp2pp2dp2 --no-cpu-baseline
run ref_cfg3 --impl reference --workload gpt3-6.7b-tp4pp2-to-tp2pp2dp2 --steps 3 --warmup 3
run cfg4 --workload gpt3-6.7b-recovery --no-cpu-baseline
run ref_cfg4 --impl reference --workload gpt3-6.7b-recovery --steps 3 --warmup 3
run dataset --workload dataset-100m-dp2to4to8
run ref_dataset --impl reference --workload dataset-100m-dp2to4to8 --steps 3 --warmup 3
run central --mode central --no-cpu-baseline
for n in 2 4 8; do RESHARD_SAME_GPU=1 run emu_n$n --gpus $n --no-cpu-baseline; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-digests > $O/launches.out 2>&1; echo launches rc=$?
timeout 900 ncu --kernel-name regex:"repart" --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_k5.csv python bench.py --workload dataset-100m-dp2to4to8 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/launches_k5.out 2>&1; echo launches_k5 rc=$?

timeout 1500 python scripts/stress_dataset.py --cases 2000 --seed 2048 > $O/stress_dataset.jsonl 2> $O/stress_dataset.err; tail -1 $O/stress_dataset.jsonl
for w in gpt3-1.3b-dp-scaleout gpt3-6.7b-tp4pp2-to-tp2pp2dp2 gpt3-6.7b-recovery; do
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:copy_bulk_dyn -s 3 -c 1 -o $O/full_$w python bench.py --workload $w --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-digests > $O/ncu_$w.out 2>&1; tail -1 $O/ncu_$w.out | cut -c1-150
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:copy_bulk_strided -s 3 -c 1 -o $O/full_gpt2-small-tp2-to-pp2 python bench.py --workload gpt2-small-tp2-to-pp2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-digests > $O/ncu_gpt2.out 2>&1; tail -1 $O/ncu_gpt2.out | cut -c1-150
