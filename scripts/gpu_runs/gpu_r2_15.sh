#!/bin/bash
# round 2, call 15: host-buffer paths on one GPU (chunked run_host vs the world pipeline), K sweep
O=gpurun_out/r2_15; mkdir -p $O
for c in 32 64 128 256; do RESHARD_HOST_CHUNKS=$c timeout 600 python scripts/probe_world_e2e.py > $O/world_e2e_$c.json 2> $O/world_e2e_$c.err; echo "chunks=$c $(cat $O/world_e2e_$c.json)"; tail -2 $O/world_e2e_$c.err; done
