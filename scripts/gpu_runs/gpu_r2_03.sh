#!/bin/bash
# round 2, call 3: new parity tests (K3T tensor maps, digests, full-size 6.7B), K5 load-flavour
# A/B with sector counters, K3T vs per-row bulk A/B on configs 1 and 3
O=gpurun_out/r2_03; mkdir -p $O
python -m pytest tests/test_full_size.py tests/test_gpu_executor.py tests/test_checkpoint.py tests/test_dataset.py -m gpu -x -q > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt
for ld in ldg v4na cg; do
  RESHARD_K5_LOAD=$ld timeout 600 python bench.py --workload dataset-100m-dp2to4to8 --no-cpu-baseline --no-e2e > $O/ds_$ld.json 2> $O/ds_$ld.err
  python -c "import json;d=json.load(open('$O/ds_$ld.json'));print('$ld',d['value'],d['roofline']['kernel_ms_per_step'],d['roofline']['gather_write_floor_ms'],d['spot_check'])"
  RESHARD_K5_LOAD=$ld timeout 600 ncu --kernel-name regex:"repart_gather2" --launch-count 2 --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed \
    --csv --log-file $O/k5_$ld.csv python bench.py --workload dataset-100m-dp2to4to8 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/k5_ncu_$ld.out 2>&1
done
for w in gpt2-small-tp2-to-pp2 gpt3-6.7b-tp4pp2-to-tp2pp2dp2 gpt3-1.3b-dp-scaleout; do
  for t in 0 1; do
    RESHARD_TMA_TENSOR=$t timeout 900 python bench.py --workload $w --no-cpu-baseline --no-e2e > $O/k3t_${w}_$t.json 2> $O/k3t_${w}_$t.err
    python -c "import json;d=json.load(open('$O/k3t_${w}_$t.json'));print('$w tensor=$t',d['value'],d['ms_min'],d['roofline']['frac'],d['verify_mismatched_bytes'],d['host_ms'])"
  done
done
