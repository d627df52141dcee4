#!/usr/bin/env python
"""K8 window sweep on the GPU: the windowed parallel Fisher-Yates at several window sizes
(RESHARD_K8_WINDOW), each checked bit-identical to the host shuffle_epoch and timed (median of
5 after 2 warm-ups).  One JSON line per window.  (r67 also ran the retired full-active-set
variant, RESHARD_K8=full, as the first line.)

    python scripts/probe_k8.py [--n N] [--fracs 80,40,20]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_05181_b200 as rs  # noqa: E402


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100_000_000)
    ap.add_argument("--fracs", default="20,40,80,100,160", help="windows as N / f")
    args = ap.parse_args()
    n, seed, ep = args.n, 0x5EED, 3
    ctx = rs.Context(1, [0], [0])
    want = rs.shuffle_epoch(n, seed, ep)
    d = ctx.malloc(0, 8 * n)
    got = np.empty(n, np.uint64)
    for f in map(int, args.fracs.split(",")):  # 0: the default window
        w = n // f if f else "default"
        if f:
            os.environ["RESHARD_K8_WINDOW"] = str(w)
        else:
            os.environ.pop("RESHARD_K8_WINDOW", None)
        ts = [rs.shuffle_epoch_device(ctx, 0, n, seed, ep, d) for _ in range(7)][2:]
        ctx.dtoh(0, got.ctypes.data, d, 8 * n)
        print(json.dumps({"window": w, "n": n, "ms_median": round(statistics.median(t["ms"] for t in ts), 3),
                          "ms_min": round(min(t["ms"] for t in ts), 3), "rounds": ts[-1]["rounds"],
                          "launches": ts[-1]["launches"], "bit_identical": bool(np.array_equal(got, want))}), flush=True)
    ctx.free(0, d)
    return 0


if __name__ == "__main__":
    sys.exit(main())
