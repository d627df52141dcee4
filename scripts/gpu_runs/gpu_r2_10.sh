#!/bin/bash
# round 2, call 10: DRAM partition balance (min / max dram__cycles_active per instance) of a plain
# torch copy vs our copy kernels on the default workload
O=gpurun_out/r2_10; mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__cycles_active.avg.pct_of_peak_sustained_elapsed,dram__cycles_active.min.pct_of_peak_sustained_elapsed,dram__cycles_active.max.pct_of_peak_sustained_elapsed
timeout 600 ncu --metrics $M --print-metric-instances values --clock-control none -s 2 -c 1 --csv --log-file $O/torch_copy.csv python scripts/probe_torch_copy.py > $O/torch.out 2>&1; tail -1 $O/torch.out
timeout 600 ncu --metrics $M --print-metric-instances values --clock-control none -k regex:copy_bulk_strided -s 3 -c 1 --csv --log-file $O/bulk.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/bulk.out 2>&1; tail -1 $O/bulk.out | cut -c1-100
RESHARD_COPY_KERNEL=ldg timeout 600 ncu --metrics $M --print-metric-instances values --clock-control none -k regex:copy_v16 -s 3 -c 1 --csv --log-file $O/ldg.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ldg.out 2>&1; tail -1 $O/ldg.out | cut -c1-100
