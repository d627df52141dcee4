#!/bin/bash
# round 2, call 28 (re-created container): GPU suite, smoke and the default line on the rebuilt tree
O=gpurun_out/r2_28; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt; grep -E "FAILED" $O/pytest.txt | head
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -2 $O/smoke.txt
timeout 1200 python bench.py > $O/default.json 2> $O/default.err; echo default rc=$?; tail -c 600 $O/default.json
