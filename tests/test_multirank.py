"""Host-side logic of the one-process-per-GPU path on CPU (gloo, world_size 2): every rank
builds the same plan and layout independently, the ranks agree on all arena sizes, and the
union of the per-rank tile lists (push: a GPU executes the fragments it holds) covers the
plan's bytes exactly once."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, workload, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        import paper_2312_05181_b200 as rs

        cat, a, b, plan, src_gpu, dst_gpu = bench.build_plan(rs, workload, world)
        ctx = rs.Context(world, [], [])  # planning-only: this CPU box has no GPU
        ex = rs.Executor(ctx, plan, src_gpu, dst_gpu, 256 << 10)
        mine = {"arenas": [ex.arena_bytes(g) for g in range(world)], "tiles": ex.tiles(rank),
                "stats": plan.stats(), "text_hash": rs.fnv1a64(plan.text().encode())}
        everyone = [None] * world
        dist.all_gather_object(everyone, mine)
        q.put((rank, everyone))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("workload", ["gpt2-small-tp2-to-pp2", "gpt3-1.3b-dp-scaleout"])
def test_two_ranks_agree_on_layout_and_cover_plan(workload):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, workload, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    views = results[0]
    assert results[1] == views  # identical gathered views on both ranks
    assert views[0]["arenas"] == views[1]["arenas"] and views[0]["text_hash"] == views[1]["text_hash"]
    st = views[0]["stats"]
    total = sum(v["tiles"][1] for v in views)
    assert total == st["moved_bytes"] + st["relayout_bytes"]
    # dst arenas hold exactly the non-kept destination bytes (plus 256-byte alignment)
    dst = sum(views[0]["arenas"][g][1] for g in range(world))
    assert st["dst_bytes"] - st["kept_bytes"] <= dst <= st["dst_bytes"] - st["kept_bytes"] + 256 * 20000
