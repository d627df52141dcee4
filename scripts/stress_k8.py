#!/usr/bin/env python
"""GPU stress of K8 (shuffle_epoch_device) against the host Fisher-Yates loop: random
(n, seed, epoch) with n log-uniform in [1, 4M] and, half the time, a random window
(RESHARD_K8_WINDOW, down to n/2000) so that the carried-list, fresh-window and graph-batch
boundaries are hit in every combination.

    python scripts/stress_k8.py [--cases N] [--seed S] > stress_k8.jsonl
"""
from __future__ import annotations

import argparse
import json
import math
import os
import random
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_05181_b200 as rs  # noqa: E402


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=3000)
    ap.add_argument("--seed", type=int, default=8)
    args = ap.parse_args()
    rng = random.Random(args.seed)
    ctx = rs.Context(1, [0], [0])
    cap = 4_000_000
    d = ctx.malloc(0, 8 * cap)
    got = np.empty(cap, np.uint64)
    t0, total, rounds = time.time(), 0, 0
    for case in range(args.cases):
        n = max(1, int(math.exp(rng.uniform(0, math.log(cap)))))
        seed, ep = rng.getrandbits(64), rng.randint(0, 1000)
        if rng.random() < 0.5:
            os.environ["RESHARD_K8_WINDOW"] = str(rng.randint(max(1, n // 2000), max(1, n)))
        else:
            os.environ.pop("RESHARD_K8_WINDOW", None)
        t = rs.shuffle_epoch_device(ctx, 0, n, seed, ep, d)
        ctx.dtoh(0, got.ctypes.data, d, 8 * n)
        if not np.array_equal(got[:n], rs.shuffle_epoch(n, seed, ep)):
            print(json.dumps({"error": "K8 differs", "n": n, "seed": seed, "epoch": ep,
                              "window": os.environ.get("RESHARD_K8_WINDOW")}), flush=True)
            return 1
        total += n
        rounds += t["rounds"]
        if (case + 1) % 500 == 0:
            print(json.dumps({"cases": case + 1, "elements": total, "rounds": rounds, "s": round(time.time() - t0, 1)}),
                  flush=True)
    print(json.dumps({"summary": "all bit-identical to the host loop", "cases": args.cases, "elements": total,
                      "rounds": rounds, "seconds": round(time.time() - t0, 1)}), flush=True)
    ctx.free(0, d)
    return 0


if __name__ == "__main__":
    sys.exit(main())
