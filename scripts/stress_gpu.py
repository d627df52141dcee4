#!/usr/bin/env python
"""GPU stress run of the apply_plan data plane (beyond the suite's 200 transitions): random
catalogs (rank 1-3, all dtypes, TP dims or replicated, up to 8 layers), random (T,P,D) pairs
including fresh destination devices and failure recovery, random tile sizes, every copy
kernel (K3T tensor-map tiles on or off), DP up to 8 (fan-out groups beyond kMaxFan), and
single-process worlds of 1, 2, 4 or 8 GPUs mapped onto cuda:0 (peer tiles, K2 fan-out with
mixed local / remote replicas, TMA peer stores on or off); every 10th case also checks the
ExecutionReport digests (destination == source == the oracle's base-tensor FNV).  Every destination cell is
compared with the oracle's apply_plan (bytes moved by the reference's slice / merge).

    python scripts/stress_gpu.py [--cases N] [--seed S] > stress.jsonl
Prints one JSON line per 100 cases and a summary line; exits 1 on the first mismatch.
"""
from __future__ import annotations

import argparse
import json
import os
import random
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2312_05181_b200 as rs  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402  (the checker)

KERNELS = ["bulk_strided", "bulk", "ldg", "bulk_dyn"]


def entries(rng):
    ent = []
    for i in range(rng.randint(1, 8)):
        rank = rng.choice([1, 2, 2, 3])
        shape = tuple(rng.choice([2, 4, 6, 8, 12, 24, 48]) for _ in range(rank))
        ent.append((f"t{i}", rng.choice([0, 1, 2, 3]), shape, rng.choice([-1] + list(range(rank))), i))
    return ent


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=2000)
    ap.add_argument("--seed", type=int, default=20260)
    args = ap.parse_args()
    rng = random.Random(args.seed)
    orc = Oracle()
    cfgs = [(T, P, D) for T in (1, 2, 3, 4, 8) for P in (1, 2, 3) for D in (1, 2, 4, 8) if T * P * D <= 8]
    ctxs = {w: rs.Context(w, list(range(w)), [0] * w) for w in (1, 2, 4, 8)}
    done, cells, t0 = 0, 0, time.time()
    stats = {"recovery": 0, "fresh": 0, "bulk_peer": 0, "tma_tensor": 0, "fanout_gt4": 0, "digest_checks": 0}
    while done < args.cases:
        ents = entries(rng)
        (T1, P1, D1), (T2, P2, D2) = rng.choice(cfgs), rng.choice(cfgs)
        if P1 > len(ents) or P2 > len(ents):
            continue
        if not all(tp < 0 or (shape[tp] % T1 == 0 and shape[tp] % T2 == 0) for _, _, shape, tp, _ in ents):
            continue
        n1, n2 = T1 * P1 * D1, T2 * P2 * D2
        failed = []
        recovery = D1 > 1 and rng.random() < 0.2
        if recovery:  # lose one whole DP replica's devices but one, re-stage onto the survivors
            victim = rng.randrange(D1)
            failed = [(0, victim * T1 * P1 + i) for i in range(T1 * P1)]
            survivors = [(0, i) for i in range(n1) if (0, i) not in failed]
            if len(survivors) < n2:
                continue
            d1, d2 = [(0, i) for i in range(n1)], survivors[:n2]
        else:
            base = rng.choice([0, 0, n1])  # sometimes fresh destination devices
            d1, d2 = [(0, i) for i in range(n1)], [(0, base + i) for i in range(n2)]
        cat, ocat = rs.Catalog.from_entries(ents), orc.catalog(ents)
        a, b = cat.build_strategy(d1, T1, P1, D1), cat.build_strategy(d2, T2, P2, D2)
        oa = ocat.build_strategy(d1, T1, P1, D1)
        ob = ocat.build_strategy(d2, T2, P2, D2)
        try:
            plan = rs.recover(a, failed, b) if failed else rs.generate_plan(a, b)
        except rs.ReshardError as e:
            if e.name == "CheckpointRequired":
                continue
            raise
        oplan = oa.plan(ob, failed=list(failed))
        if plan.text() != oplan.text():
            print(json.dumps({"error": "plan text differs", "case": done}), flush=True)
            return 1
        world = rng.choice([1, 1, 2, 4, 8])
        os.environ["RESHARD_COPY_KERNEL"] = rng.choice(KERNELS)
        peer = rng.random() < 0.3
        os.environ["RESHARD_BULK_PEER"] = "1" if peer else "0"
        tensor = rng.random() < 0.3  # K3T: strided pieces as TMA tensor boxes (bulk_strided only)
        os.environ["RESHARD_TMA_TENSOR"] = "1" if tensor else "0"
        ctx = ctxs[world]
        # logical device -> world GPU: the device ordinal's index in the layout, mod world
        all_devs = sorted(set(d1) | set(d2))
        gpu = {d: i % world for i, d in enumerate(all_devs)}
        ex = rs.Executor(ctx, plan, [gpu[d] for d in d1], [gpu[d] for d in d2], rng.choice([4096, 65536, 256 << 10]))
        ex.allocate_local()
        ex.prepare()
        ex.fill_sources()
        ex.apply()
        if ex.verify() != 0:
            print(json.dumps({"error": "verify mismatch", "case": done}), flush=True)
            return 1
        if done % 10 == 0:  # ExecutionReport digests: destination == source == oracle
            dd, sd = ex.digests(1, replica=-1), ex.digests(0)
            if dd != sd or any(dd[t] != ocat.base_digest(t) for t in dd):
                print(json.dumps({"error": "digest mismatch", "case": done}), flush=True)
                return 1
            stats["digest_checks"] += 1
        ost, _ = oplan.apply(oa.fill(), n_threads=4)
        for dev, t, c, bnd in ex.dst_cells():
            got = np.zeros(bnd.nbytes, np.uint8)
            ctx.dtoh(0, got.ctypes.data, ex.cell_ptr(bnd), bnd.nbytes)
            if not np.array_equal(got, ost.cell(d2[dev], t, b.cell(t, c))):
                print(json.dumps({"error": "cell mismatch", "case": done, "tensor": t, "cell": c}), flush=True)
                return 1
            cells += 1
        del ex
        stats["recovery"] += recovery
        stats["fresh"] += (not recovery) and d2[0][1] >= n1
        stats["bulk_peer"] += peer and world > 1
        stats["tma_tensor"] += tensor and os.environ["RESHARD_COPY_KERNEL"] in ("bulk_strided", "bulk_dyn")
        stats["fanout_gt4"] += D2 > 4
        done += 1
        if done % 100 == 0:
            print(json.dumps({"cases": done, "cells": cells, "s": round(time.time() - t0, 1)}), flush=True)
    print(json.dumps({"summary": "all byte-exact", "cases": done, "cells": cells, **stats,
                      "seconds": round(time.time() - t0, 1)}), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
