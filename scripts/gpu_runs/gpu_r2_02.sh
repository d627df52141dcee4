#!/bin/bash
# round 2, call 2: full-size 6.7B parity, prepare trace, 6.7B bench lines + CPU reference arms,
# K5 sector counters (default vs 32-byte L2 fetch granularity)
O=gpurun_out/r2_02; mkdir -p $O
python -m pytest tests/test_full_size.py tests/test_checkpoint.py -m gpu -x -q > $O/pytest_full.txt 2>&1; tail -3 $O/pytest_full.txt
RESHARD_HOST_TRACE=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 > $O/bench_trace.json 2> $O/bench_trace.err; grep prepare-trace $O/bench_trace.err | head; python -c "import json;d=json.load(open('$O/bench_trace.json'));print(d['value'],d['host_ms'])"
for w in gpt3-6.7b-tp4pp2-to-tp2pp2dp2 gpt3-6.7b-recovery; do
  timeout 1200 python bench.py --workload $w --no-cpu-baseline --steps 10 > $O/bench_$w.json 2> $O/bench_$w.err; python -c "import json;d=json.load(open('$O/bench_$w.json'));print('$w',d['value'],d['waves'],d['roofline']['frac'],d['verify_mismatched_bytes'],d['host_ms'],d['e2e'])"; tail -2 $O/bench_$w.err
  timeout 1200 python bench.py --impl reference --workload $w --steps 2 --warmup 3 > $O/ref_$w.json 2> $O/ref_$w.err; tail -c 600 $O/ref_$w.json; tail -2 $O/ref_$w.err
done
for f in default 32; do
  if [ $f = 32 ]; then export RESHARD_L2_FETCH=32; fi
  timeout 900 ncu --kernel-name regex:"repart_gather2|gather_write_probe|gather_probe" --launch-count 6 --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__sectors_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_requests_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex_lookup_miss.sum \
    --csv --log-file $O/k5_sectors_$f.csv python bench.py --workload dataset-100m-dp2to4to8 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/k5_ncu_$f.out 2>&1
  tail -2 $O/k5_ncu_$f.out
done
