#!/usr/bin/env python
"""rs_broadcast on one B200: 1 GiB to k = 1..8 destinations (all on cuda:0), event time and
HBM bytes (one read per group of 4 destinations + k writes) against the measured HBM peak."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2312_05181_b200 as rs  # noqa: E402

ctx = rs.Context(1, [0], [0])
n = 1 << 30
src = ctx.malloc(0, n)
dsts = [ctx.malloc(0, n) for _ in range(8)]
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
for k in (1, 2, 4, 8):
    ts = [rs.broadcast(ctx, 0, src, dsts[:k], n) for _ in range(6)][1:]
    ms = min(t["ms"] for t in ts)
    traffic = ts[0]["read_bytes"] + ts[0]["bytes"]
    print(json.dumps({"destinations": k, "bytes": n, "ms": round(ms, 3), "hbm_gbs": round(traffic / ms / 1e6, 1),
                      "frac_of_peak": round(traffic / ms / 1e6 / peak, 3)}), flush=True)
