#!/usr/bin/env python
"""SPEC acceptance #10 (process / in-process equivalence): the paper's §6.2 elastic
sequence (TP,PP,DP) = (2,4,2) -> (2,4,1) -> (2,2,1), and back to (2,4,2) (re-staging plus a DP
fan-out over peers), on a toy GPT, executed as a CHAIN — each
reconfiguration's destination cells are the next one's sources — in either worker mode:

  in-process:  python scripts/elastic_sequence.py --world W          (one process drives W GPUs)
  process:     torchrun --nproc-per-node W scripts/elastic_sequence.py --world W
               (one process per GPU, CUDA-IPC destination arenas, gloo plumbing)

Logical device d of every layout sits on world GPU d % W (RESHARD_SAME_GPU=1 maps every world
GPU onto cuda:0).  Only the first layout is filled (K6 synthetic payload); every later step
reads what the previous one wrote.  After each step every destination byte is checked against
the regenerated base-tensor payload (K7), and rank 0 prints one JSON line with the per-step
plan / executed byte counts and the FNV-1a-64 digest of every destination cell of every step —
the two modes must print identical lines (tests/test_gpu_multiprocess.py)."""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2312_05181_b200 as rs  # noqa: E402

SEQUENCE = [(2, 4, 2), (2, 4, 1), (2, 2, 1), (2, 4, 2)]  # §6.2 (T, P, D), then back to the start


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=4)
    ap.add_argument("--tile-kib", type=int, default=16)
    args = ap.parse_args()
    W = args.world
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    dist = None
    if world > 1:
        import torch.distributed as dist

        if world != W:
            raise SystemExit(f"--world {W} but WORLD_SIZE={world}")
        dist.init_process_group("gloo")
        mine = [rank]
    else:
        mine = list(range(W))
    cuda_of = [0] * len(mine) if os.environ.get("RESHARD_SAME_GPU") else mine
    ctx = rs.Context(W, mine, cuda_of)

    cat = rs.Catalog.gpt(64, 8, 16, 128, rs.MIXED_ADAM)
    layouts = []
    for t, p, d in SEQUENCE:
        devs = [(0, i) for i in range(t * p * d)]
        layouts.append(cat.build_strategy(devs, t, p, d))

    def barrier():
        for g in mine:
            ctx.sync(g)
        if dist is not None:
            dist.barrier()

    steps, prev, owned = [], None, []
    for s in range(len(layouts) - 1):
        a, b = layouts[s], layouts[s + 1]
        plan = rs.generate_plan(a, b)
        ex = rs.Executor(ctx, plan, [i % W for i in range(len(a.devices))], [i % W for i in range(len(b.devices))],
                         args.tile_kib << 10)
        ptrs = {}
        for g in mine:
            sb, db = ex.arena_bytes(g)
            ptrs[g] = (ctx.malloc(g, max(sb, 256)), ctx.malloc(g, max(db, 256)))
            owned += [(g, ptrs[g][0]), (g, ptrs[g][1])]
            ex.bind(g, *ptrs[g])
        if dist is not None:  # every GPU's destination arena, mapped into this process
            handles = [None] * world
            dist.all_gather_object(handles, ctx.ipc_handle(rank, ptrs[rank][1]))
            for g in range(world):
                if g != rank:
                    ex.bind(g, 0, ctx.ipc_open(rank, handles[g]))
        ex.prepare()
        if prev is None:
            ex.fill_sources()
        else:  # this step's sources = the previous step's destination cells (same device -> GPU map)
            where = {}
            for dev, t, c, bnd in prev.dst_cells():
                where[(dev, t, tuple(map(tuple, a.cell(t, c))))] = bnd
            src = ex.src_cells()
            k = 0
            for i, dev in enumerate(a.devices):
                for t, box in a.hosted_subtensors(dev):
                    bnd = src[k]
                    k += 1
                    if bnd.gpu not in mine or bnd.nbytes == 0:
                        continue
                    pb = where[(i, t, tuple(map(tuple, box)))]
                    buf = np.empty(bnd.nbytes, np.uint8)
                    ctx.dtoh(bnd.gpu, buf.ctypes.data, prev.cell_ptr(pb), bnd.nbytes)
                    ctx.htod(bnd.gpu, ex.cell_ptr(bnd), buf.ctypes.data, bnd.nbytes)
            assert k == len(src)
        barrier()
        ex.run()
        t = ex.wait()
        barrier()
        bad = ex.verify()
        digests = {}
        for dev, tt, c, bnd in ex.dst_cells():
            if bnd.gpu in mine and bnd.nbytes:
                buf = np.empty(bnd.nbytes, np.uint8)
                ctx.dtoh(bnd.gpu, buf.ctypes.data, ex.cell_ptr(bnd), bnd.nbytes)
                digests[f"{dev}/{tt}/{c}"] = f"{rs.fnv1a64(buf.tobytes()):016x}"
        st = plan.stats()
        local = {"bad": bad, "bytes": sum(x["bytes"] for x in t), "digests": digests}
        if dist is not None:
            allv = [None] * world
            dist.all_gather_object(allv, local)
        else:
            allv = [local]
        steps.append({"from": list(SEQUENCE[s]), "to": list(SEQUENCE[s + 1]), "plan_text_fnv": f"{rs.fnv1a64(plan.text().encode()):016x}",
                      "moved_bytes": st["moved_bytes"], "relayout_bytes": st["relayout_bytes"],
                      "n_move": st["n_move"], "n_merge": st["n_merge"], "n_split": st["n_split"],
                      "executed_bytes": sum(v["bytes"] for v in allv), "mismatched_bytes": sum(v["bad"] for v in allv),
                      "digests": dict(sorted(kv for v in allv for kv in v["digests"].items()))})
        barrier()
        prev = ex
    if rank == 0:
        print(json.dumps({"world": W, "mode": "process" if dist is not None else "in-process", "steps": steps}), flush=True)
    barrier()
    for g, p in owned:
        ctx.free(g, p)
    return 0


if __name__ == "__main__":
    sys.exit(main())
