#!/usr/bin/env python
"""GPU stress run of the dataset path (K5 repartition + locate, K8 shuffle) against the
oracle's restatement: random corpus sizes (1 .. 2M samples, 1 .. 300 files,
variable lengths), global batches, DP changes and at_steps (trailing partial batches,
at_step 0, the last batch), every rank, both index layouts, every K5 variant, the multi-rank
batch (fused and two-stream) over 1-3 DP events; and random
(n, seed, epoch) for the GPU Fisher-Yates.

    python scripts/stress_dataset.py [--cases N] [--seed S] > stress_dataset.jsonl
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


def corpus(n, n_files, rng):
    per = (n + n_files - 1) // n_files
    files = np.arange(n, dtype=np.uint64) // np.uint64(per)
    lens = np.frombuffer(rng.randbytes(4 * n), np.uint32).astype(np.uint64) % np.uint64(9000) + np.uint64(1)
    offs = np.zeros(n, np.uint64)
    starts = np.searchsorted(files, np.arange(n_files, dtype=np.uint64))
    cs = np.cumsum(lens) - lens
    offs = cs - cs[starts[files.astype(np.int64)]]
    return np.stack([files, offs.astype(np.uint64), lens], axis=1).copy()


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=500)
    ap.add_argument("--seed", type=int, default=99)
    args = ap.parse_args()
    rng = random.Random(args.seed)
    orc = Oracle()
    ctx = rs.Context(1, [0], [0])
    t0, ranks, samples_checked, batched_ranks = time.time(), 0, 0, 0
    modes = ["split2", "split2", "split2_6", "lookback"]
    for case in range(args.cases):
        n = rng.choice([1, 7, 100, 1000, 4096, 65_537, 300_000, 1_000_003, 2_000_000])
        nf = rng.randint(1, 300)
        dp_new = rng.choice([1, 2, 3, 4, 5, 8])
        B = dp_new * rng.randint(1, 96)
        full = n // B
        at = rng.choice([0, full // 2, max(full - 1, 0), full]) if full else 0
        samples = corpus(n, nf, rng)
        perm = rs.shuffle_epoch(n, rng.getrandbits(32), rng.randint(0, 9))
        if case % 10 == 0:  # K8 against the host loop on the same (n, seed, epoch) family
            seed, ep = rng.getrandbits(32), rng.randint(0, 9)
            d_p = ctx.malloc(0, 8 * n)
            rs.shuffle_epoch_device(ctx, 0, n, seed, ep, d_p)
            got = np.empty(n, np.uint64)
            ctx.dtoh(0, got.ctypes.data, d_p, 8 * n)
            ctx.free(0, d_p)
            if not np.array_equal(got, rs.shuffle_epoch(n, seed, ep)):
                print(json.dumps({"error": "K8 differs", "n": n}), flush=True)
                return 1
        mode = rng.choice(modes)
        eb = 24 if mode == "lookback" else rng.choice([24, 32])
        os.environ["RESHARD_K5"] = mode
        d_perm, d_samp = ctx.malloc(0, 8 * n), ctx.malloc(0, 24 * n)
        ctx.htod(0, d_perm, perm.ctypes.data, 8 * n)
        ctx.htod(0, d_samp, samples.ctypes.data, 24 * n)
        d_idx = d_samp
        if eb == 32:
            d_idx = ctx.malloc(0, 32 * n)
            rs.dataset_index_pad(ctx, 0, d_samp, d_idx, n)
        # every other case: the ranks of 1-3 DP events of this corpus as ONE rs_repartition_batch
        # (fused one-launch-per-pass, or the two-stream schedule), else one rs_repartition per rank
        batch = mode.startswith("split2") and case % 2 == 1
        fuse = rng.choice(["1", "0"])
        os.environ["RESHARD_K5_FUSE"] = fuse
        events = [(at, dp_new)]
        if batch:
            for _ in range(rng.randint(0, 2)):
                dp2 = rng.choice([dd for dd in (1, 2, 3, 4, 5, 8) if B % dd == 0])
                events.append((rng.choice([0, full // 3, full]) if full else 0, dp2))
        try:
            jobs = []
            for at_e, dp_e in events:
                for d in range(dp_e):
                    fc = np.array([rng.choice([0, 1, 2]) for _ in range(nf)], np.uint8)
                    d_fc = ctx.malloc(0, nf)
                    ctx.htod(0, d_fc, fc.ctypes.data, nf)
                    cnt = rs.repartition_count(n, B, at_e, dp_e, d)
                    jobs.append((at_e, dp_e, d, d_fc, rs.Partition(ctx, 0, cnt), fc))
            if batch:
                rs.repartition_batch(ctx, 0, d_perm, d_idx, n, B, [j[:5] for j in jobs], entry_bytes=eb)
            else:
                for at_e, dp_e, d, d_fc, part, _ in jobs:
                    rs.repartition(ctx, 0, d_perm, d_idx, d_fc, n, B, at_e, dp_e, d, part, entry_bytes=eb)
            for at_e, dp_e, d, d_fc, part, fc in jobs:
                got = part.fetch()
                want = orc.dataset_gather(n, B, at_e, dp_e, d, perm, samples, fc, n_threads=8)
                for key in ("pos", "ent", "boff", "qidx"):
                    if not np.array_equal(got[key], want[key]):
                        print(json.dumps({"error": f"{key} differs", "n": n, "B": B, "at": at_e, "dp": dp_e, "d": d,
                                          "mode": mode, "eb": eb, "batch": batch, "fuse": fuse}), flush=True)
                        return 1
                if got["qcount"] != want["qcount"]:
                    print(json.dumps({"error": "qcount differs", "n": n, "batch": batch, "fuse": fuse}), flush=True)
                    return 1
                part.free()
                ctx.free(0, d_fc)
                ranks += 1
                samples_checked += part.count
                batched_ranks += 1 if batch else 0
        finally:
            for p in (d_perm, d_samp) + ((d_idx,) if eb == 32 else ()):
                ctx.free(0, p)
        if (case + 1) % 50 == 0:
            print(json.dumps({"cases": case + 1, "ranks": ranks, "samples": samples_checked,
                              "s": round(time.time() - t0, 1)}), flush=True)
    print(json.dumps({"summary": "all equal to the oracle", "cases": args.cases, "ranks": ranks,
                      "ranks_in_batches": batched_ranks, "samples": samples_checked,
                      "seconds": round(time.time() - t0, 1)}), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
