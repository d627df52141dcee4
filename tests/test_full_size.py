"""BASELINE configs[2] and configs[3] at FULL size on one B200: GPT-3 6.7B
model + Adam state (93.2 GB) resharded (TP4,PP2,DP1)->(TP2,PP2,DP2) and recovered
(TP2,PP2,DP2)->(TP2,PP2,DP1) after losing devices {1,3,4,6}.  All logical
devices live on cuda:0; a plan larger than its HBM runs in catalog windows (waves) over reused
arenas.  Every destination byte is checked by K7 (regenerate-and-compare of the splitmix64
payload, kernels.cu verify) and sampled destination cells are compared byte for byte with the
oracle's own generation of that box of the base tensor (a destination cell is slice(base, cell),
proj/src/tensor/tensor.cpp:61-78)."""
import random

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _waves_that_fit(rs, bench, cat, plan, src_gpu, dst_gpu):
    import torch

    free, _ = torch.cuda.mem_get_info(0)
    pctx = rs.Context(1, [], [])
    for waves in range(1, 9):
        wins = bench.windows_of(cat, waves)
        pex = [rs.Executor(pctx, plan, src_gpu, dst_gpu, window=w if len(wins) > 1 else None) for w in wins]
        need = max(sum(p.arena_bytes(0)) for p in pex)
        if need <= 0.9 * free:
            return wins
    raise AssertionError("no wave count fits")


@pytest.mark.parametrize("workload", ["gpt3-6.7b-tp4pp2-to-tp2pp2dp2", "gpt3-6.7b-recovery"])
def test_gpt3_67b_full_size(rs, orc, ctx, workload):
    import bench

    cat, a, b, plan, src_gpu, dst_gpu = bench.build_plan(rs, workload, 1)
    st = plan.stats()
    if workload.endswith("recovery"):
        assert round(st["moved_bytes"] / 1e9, 2) == 46.67
        assert st["n_merge"] == 0
    else:
        assert (st["n_move"], st["n_merge"]) == (6964, 3088)
        assert round(st["moved_bytes"] / 1e9, 2) == 163.17
    (h, L, S, V, kind), *_ = bench.WORKLOADS[workload]
    ocat = orc.catalog_gpt(h, L, S, V, kind)
    wins = _waves_that_fit(rs, bench, cat, plan, src_gpu, dst_gpu)
    if workload.endswith("recovery"):
        assert len(wins) == 1  # failed devices hold no state: the recovery fits one wave
    rng = random.Random(7)
    checked, cells, total = 0, 0, 0
    for w in wins:
        ex = rs.Executor(ctx, plan, src_gpu, dst_gpu, window=w if len(wins) > 1 else None)
        ex.allocate_local()
        ex.prepare()
        ex.fill_sources()
        t = ex.apply()
        total += t[0]["bytes"]
        assert ex.verify() == 0, f"K7 mismatches in window {w}"
        mine = [x for x in ex.dst_cells() if w[0] <= x[1] < w[1] and x[3].gpu == 0]
        cells += len(mine)
        small = [x for x in mine if x[3].nbytes <= (96 << 20)]
        for dev, tt, c, bnd in rng.sample(small, min(6, len(small))):
            got = np.zeros(bnd.nbytes, np.uint8)
            ctx.dtoh(0, got.ctypes.data, ex.cell_ptr(bnd), bnd.nbytes)
            want = ocat.box_bytes(tt, b.cell(tt, c))
            assert np.array_equal(got, want), f"tensor {tt} cell {c} of device {dev}"
            checked += 1
        del ex
    assert checked >= 6 and cells > 0
    assert total == st["moved_bytes"] + st["relayout_bytes"]  # every algorithmic byte written once
