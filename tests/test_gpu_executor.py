"""GPU parity of the apply_plan data plane: every destination cell produced by the sm_100a
tile kernel, read back through the C-ABI, must equal the oracle's apply_plan result
(bytes moved by the reference's slice/merge, tensor.cpp:61-114) byte for byte."""
import ctypes
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DEV = lambda n, w=0: [(w, i) for i in range(n)]  # noqa: E731


def _run(rs, ctx, plan, n_src, n_dst, tile=256 << 10):
    ex = rs.Executor(ctx, plan, [0] * n_src, [0] * n_dst, tile)
    ex.allocate_local()
    ex.prepare()
    ex.fill_sources()
    t = ex.apply()
    return ex, t


def _compare_with_oracle(rs, ctx, ex, b_ptc, ostate, devs):
    n = 0
    for dev, t, c, bnd in ex.dst_cells():
        got = np.zeros(bnd.nbytes, np.uint8)
        ctx.dtoh(0, got.ctypes.data, ex.cell_ptr(bnd), bnd.nbytes)
        want = ostate.cell(devs[dev], t, b_ptc.cell(t, c))
        assert np.array_equal(got, want), f"tensor {t} cell {c} on device {devs[dev]}"
        n += 1
    return n


def _pair(rs, orc, entries, a_cfg, b_cfg, failed=()):
    cat = rs.Catalog.from_entries(entries)
    ocat = orc.catalog(entries)
    (T1, P1, D1, d1), (T2, P2, D2, d2) = a_cfg, b_cfg
    a, b = cat.build_strategy(d1, T1, P1, D1), cat.build_strategy(d2, T2, P2, D2)
    oa, ob = ocat.build_strategy(d1, T1, P1, D1), ocat.build_strategy(d2, T2, P2, D2)
    plan = rs.recover(a, failed, b) if failed else rs.generate_plan(a, b)
    oplan = oa.plan(ob, failed=list(failed))
    assert plan.text() == oplan.text()
    return a, b, plan, oa, ob, oplan


def test_fig6_end_to_end(rs, orc, ctx):
    entries = [("t1", 0, (6,), 0, 0), ("t2", 0, (6,), 0, 1)]
    a, b, plan, oa, ob, oplan = _pair(rs, orc, entries, (2, 1, 1, DEV(2)), (3, 2, 1, DEV(6)))
    ex, _ = _run(rs, ctx, plan, 2, 6)
    ost, _ = oplan.apply(oa.fill(), n_threads=6)
    assert _compare_with_oracle(rs, ctx, ex, b, ost, DEV(6)) == 6
    assert ex.verify() == 0


def _random_entries(rng, n_t):
    ent = []
    for i in range(n_t):
        rank = rng.choice([1, 2, 2, 3])
        shape = tuple(rng.choice([2, 4, 6, 8, 12, 24]) for _ in range(rank))
        dtype = rng.choice([0, 1, 2, 3])
        tp = rng.choice([-1] + list(range(rank)))
        ent.append((f"t{i}", dtype, shape, tp, i))
    return ent


def _configs(n_dev_max=8):
    out = []
    for T in (1, 2, 3, 4):
        for P in (1, 2, 3):
            for D in (1, 2, 4):
                if T * P * D <= n_dev_max:
                    out.append((T, P, D))
    return out


def test_random_transitions_bytes_exact(rs, orc, ctx):
    """SPEC acceptance #1 on the GPU: random DP/TP/PP transitions, bit-identical."""
    rng = random.Random(1234)
    cfgs = _configs()
    done = 0
    while done < 200:
        n_t = rng.randint(1, 6)
        ents = _random_entries(rng, n_t)
        (T1, P1, D1), (T2, P2, D2) = rng.choice(cfgs), rng.choice(cfgs)
        if P1 > n_t or P2 > n_t:
            continue
        # TP must divide every sliced extent
        ok = all(tp < 0 or (shape[tp] % T1 == 0 and shape[tp] % T2 == 0) for _, _, shape, tp, _ in ents)
        if not ok:
            continue
        n1, n2 = T1 * P1 * D1, T2 * P2 * D2
        base = rng.choice([0, 0, n1])  # sometimes fresh destination devices
        d1, d2 = DEV(n1), [(0, base + i) for i in range(n2)]
        a, b, plan, oa, ob, oplan = _pair(rs, orc, ents, (T1, P1, D1, d1), (T2, P2, D2, d2))
        tile = rng.choice([4096, 65536, 256 << 10])
        ex, _ = _run(rs, ctx, plan, n1, n2, tile)
        ost, _ = oplan.apply(oa.fill(), n_threads=4)
        _compare_with_oracle(rs, ctx, ex, b, ost, d2)
        assert ex.verify() == 0
        done += 1


def test_gpt2_small_config1_bytes_exact(rs, orc, ctx):
    """BASELINE configs[0]: GPT-2 small fp32+Adam (TP2,PP1,DP1)->(TP1,PP2,DP1), every
    destination byte compared with the oracle running the reference's slice/merge."""
    cat = rs.Catalog.gpt(768, 12, 1024, 50304, rs.FP32_ADAM)
    a, b = cat.build_strategy(DEV(2), 2, 1, 1), cat.build_strategy(DEV(2), 1, 2, 1)
    plan = rs.generate_plan(a, b)
    ex, t = _run(rs, ctx, plan, 2, 2)
    from oracle.oracle import Oracle, lib_path
    import os

    o = Oracle(reference=os.path.exists(lib_path(True)))
    ocat = o.catalog_gpt(768, 12, 1024, 50304, 0)
    oa, ob = ocat.build_strategy(DEV(2), 2, 1, 1), ocat.build_strategy(DEV(2), 1, 2, 1)
    oplan = oa.plan(ob)
    assert oplan.text() == plan.text()
    ost, rep = oplan.apply(oa.fill(), n_threads=2)
    n = _compare_with_oracle(rs, ctx, ex, b, ost, DEV(2))
    assert n == 444
    assert ex.verify() == 0
    assert t[0]["bytes"] == rep["moved"] + rep["local"]


def test_recovery_plan_on_gpu(rs, orc, ctx):
    """configs[3] structure at toy size: (2,2,2) -> (2,2,1) on survivors, failed {1,3,4,6}."""
    h, L, S, V = 64, 4, 16, 128
    cat = rs.Catalog.gpt(h, L, S, V, rs.MIXED_ADAM)
    a = cat.build_strategy(DEV(8), 2, 2, 2)
    surv = [(0, 0), (0, 2), (0, 5), (0, 7)]
    b = cat.build_strategy(surv, 2, 2, 1)
    plan = rs.recover(a, [(0, 1), (0, 3), (0, 4), (0, 6)], b)
    st = plan.stats()
    assert st["n_split"] == 0 and st["n_merge"] == 0 and st["relayout_bytes"] == 0
    assert st["moved_bytes"] * 2 == st["dst_bytes"]
    ex, _ = _run(rs, ctx, plan, 8, 4)
    assert ex.verify() == 0


def test_gpt3_1p3b_config2_full_size(rs, ctx):
    """BASELINE configs[1] at full size (36.97 GB of destination state on one GPU):
    size-independent property check — every destination byte equals the regenerated
    base-tensor payload (K7), which the oracle pins at small sizes."""
    cat = rs.Catalog.gpt(2048, 24, 2048, 50304, rs.MIXED_ADAM)
    a, b = cat.build_strategy(DEV(2), 2, 1, 1), cat.build_strategy(DEV(4), 2, 1, 2)
    plan = rs.generate_plan(a, b)
    st = plan.stats()
    assert st["n_move"] == 2336 and st["moved_bytes"] == 18484379648
    ex, t = _run(rs, ctx, plan, 2, 4)
    assert t[0]["bytes"] == st["moved_bytes"]
    assert ex.verify() == 0


def test_device_slice_merge_vs_reference(rs, orc, ctx):
    """rs_slice / rs_merge (device) vs the oracle slice/merge on random boxes."""
    rng = random.Random(7)
    for _ in range(1000):  # acceptance #9: >= 1,000 fuzzed range queries
        rank = rng.randint(1, 4)
        shape = tuple(rng.randint(1, 9) for _ in range(rank))
        dtype = rng.choice([0, 1, 2, 3])
        w = {0: 4, 1: 2, 2: 8, 3: 1}[dtype]
        n = int(np.prod(shape)) * w
        host = np.frombuffer(rng.randbytes(n), np.uint8).copy()
        box = []
        for e in shape:
            lo = rng.randint(0, e - 1)
            box.append((lo, rng.randint(lo + 1, e)))
        want = orc.slice(dtype, shape, host, box)
        src = ctx.malloc(0, n)
        out = ctx.malloc(0, max(want.size, 1))
        ctx.htod(0, src, host.ctypes.data, n)
        rs.slice(ctx, 0, rs.DeviceTensor(dtype, shape, src), box, out)
        got = np.zeros(want.size, np.uint8)
        ctx.dtoh(0, got.ctypes.data, out, want.size)
        assert np.array_equal(got, want)
        # merge the grid cells of a random grid back
        pts = []
        for e in shape:
            k = rng.randint(0, min(2, e - 1))
            pts.append(sorted(rng.sample(range(1, e), k)) if k else [])
        cells = orc.grid_cells(shape, pts)
        parts, ptrs = [], []
        for c in cells:
            data = orc.slice(dtype, shape, host, c)
            p = ctx.malloc(0, data.size)
            ctx.htod(0, p, data.ctypes.data, data.size)
            ptrs.append(p)
            parts.append((c, rs.DeviceTensor(dtype, tuple(z - a for a, z in c), p)))
        mo = ctx.malloc(0, n)
        rs.merge(ctx, 0, parts, shape, mo)
        got = np.zeros(n, np.uint8)
        ctx.dtoh(0, got.ctypes.data, mo, n)
        assert np.array_equal(got, host)
        for p in ptrs + [src, out, mo]:
            ctx.free(0, p)


def test_device_merge_error_precedence(rs, ctx):
    """Error order of reference merge (tensor.cpp:84-98): per part check_against ->
    DtypeMismatch -> ShapeMismatch, then TilingOverlap, then TilingGap."""
    buf = ctx.malloc(0, 1024)
    T = lambda dt, sh: rs.DeviceTensor(dt, sh, buf)  # noqa: E731

    def err(parts, target):
        with pytest.raises(rs.ReshardError) as e:
            rs.merge(ctx, 0, parts, target, buf)
        return e.value.name

    assert err([], (6,)) == "TilingGap"
    assert err([([(0, 7)], T(0, (7,)))], (6,)) == "RangeOutOfBounds"
    assert err([([(0, 3), (0, 1)], T(0, (3, 1)))], (6,)) == "RankMismatch"
    assert err([([(0, 3)], T(0, (3,))), ([(3, 6)], T(1, (3,)))], (6,)) == "DtypeMismatch"
    assert err([([(0, 3)], T(0, (2,)))], (6,)) == "ShapeMismatch"
    assert err([([(0, 4)], T(0, (4,))), ([(3, 6)], T(0, (3,)))], (6,)) == "TilingOverlap"
    assert err([([(0, 3)], T(0, (3,)))], (6,)) == "TilingGap"
    # a later part's range error wins over an earlier part's dtype? no: checks are per part in order
    assert err([([(0, 3)], T(0, (3,))), ([(3, 6)], T(1, (2,))), ([(0, 9)], T(0, (9,)))], (6,)) == "DtypeMismatch"
    ctx.free(0, buf)


@pytest.mark.parametrize("min_chunk_mib", ["0", "1"])
def test_run_host_pipelined_matches_device_result(rs, ctx, min_chunk_mib, monkeypatch):
    """e2e path (host buffers, pipelined H2D / kernels / D2H): the host copy of the dst arena
    equals the device arena and every destination cell verifies — with 64 chunks of these toy
    states (no minimum chunk size) and with the chunk count capped by a 1 MiB minimum."""
    monkeypatch.setenv("RESHARD_HOST_MIN_CHUNK_MIB", min_chunk_mib)
    cat = rs.Catalog.gpt(256, 6, 64, 1024, rs.MIXED_ADAM)
    for (a_cfg, b_cfg) in [((2, 1, 1, 2), (2, 1, 2, 4)), ((2, 1, 1, 2), (1, 2, 1, 2)), ((4, 2, 1, 8), (2, 2, 2, 8))]:
        a = cat.build_strategy(DEV(a_cfg[3]), *a_cfg[:3])
        b = cat.build_strategy(DEV(b_cfg[3]), *b_cfg[:3])
        plan = rs.generate_plan(a, b)
        ex, _ = _run(rs, ctx, plan, a_cfg[3], b_cfg[3], 64 << 10)
        s_bytes, d_bytes = ex.arena_bytes(0)
        hs, hd = rs.host_alloc(s_bytes), rs.host_alloc(max(d_bytes, 1))
        src_ptr, dst_ptr = ex.arenas[0]
        ctx.dtoh(0, hs, src_ptr, s_bytes)
        ctx.memset(0, src_ptr, 0, s_bytes)  # every source byte must come from the host buffer
        ctx.memset(0, dst_ptr, 0, d_bytes)
        t = ex.run_host(0, hs, hd)
        assert t["launches"] >= 1
        assert ex.verify() == 0
        dev = np.zeros(d_bytes, np.uint8)
        ctx.dtoh(0, dev.ctypes.data, dst_ptr, d_bytes)
        host = np.ctypeslib.as_array((ctypes.c_uint8 * d_bytes).from_address(hd))
        assert np.array_equal(dev, host)
        rs.host_free(hs)
        rs.host_free(hd)


def test_run_host_skip_unread_recovery(rs, ctx, monkeypatch):
    """RS_HOST_SKIP_UNREAD on a recovery (survivors keep half of their cells in place): only the
    source ranges the tiles read cross PCIe, and every destination byte still verifies and comes
    back to the host buffer; unknown flag bits are rejected."""
    monkeypatch.setenv("RESHARD_HOST_MIN_CHUNK_MIB", "0")  # toy state: keep it multi-chunk
    cat = rs.Catalog.gpt(64, 4, 16, 128, rs.MIXED_ADAM)
    a = cat.build_strategy(DEV(8), 2, 2, 2)
    b = cat.build_strategy([(0, 0), (0, 2), (0, 5), (0, 7)], 2, 2, 1)
    plan = rs.recover(a, [(0, 1), (0, 3), (0, 4), (0, 6)], b)
    st = plan.stats()
    ex, _ = _run(rs, ctx, plan, 8, 4, 16 << 10)
    s_bytes, d_bytes = ex.arena_bytes(0)
    up_all, up_read = ex.host_upload_bytes(0), ex.host_upload_bytes(0, skip_unread=True)
    assert up_all == s_bytes
    assert up_read == st["moved_bytes"] < s_bytes  # each moved byte read once, kept cells stay home
    hs, hd = rs.host_alloc(s_bytes), rs.host_alloc(max(d_bytes, 1))
    src_ptr, dst_ptr = ex.arenas[0]
    ctx.dtoh(0, hs, src_ptr, s_bytes)
    ctx.memset(0, src_ptr, 0, s_bytes)
    ctx.memset(0, dst_ptr, 0, d_bytes)
    ex.run_host(0, hs, hd, skip_unread=True)
    # the kept cells (bound in the src arena) were not uploaded: bring them back, then every
    # destination cell — the moved ones written by the run from the uploaded ranges alone — verifies
    ctx.htod(0, src_ptr, hs, s_bytes)
    assert ex.verify() == 0
    dev = np.zeros(d_bytes, np.uint8)
    ctx.dtoh(0, dev.ctypes.data, dst_ptr, d_bytes)
    host = np.ctypeslib.as_array((ctypes.c_uint8 * d_bytes).from_address(hd))
    assert np.array_equal(dev, host)
    t = rs._capi.rs_timing()
    rc = rs.lib.rs_executor_run_host_flags(ex.h, 0, hs, hd, 6, ctypes.byref(t))
    assert rc != 0 and "flags" in rs.lib.rs_last_error().decode()
    rs.host_free(hs)
    rs.host_free(hd)


def _kat():
    import json
    import os

    return json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "tensor_core_kat.json")))


def test_reference_slice_merge_fixtures_on_device(rs, ctx):
    """The committed reference fixtures (tests/golden/tensor_core_kat.json, produced by the
    reference's own tensor.cpp) replayed through rs_slice / rs_merge on the GPU: same bytes,
    same error names — including rank-0 tensors and the error cases."""
    kat = _kat()
    W = {0: 4, 1: 2, 2: 8, 3: 1}
    buf = ctx.malloc(0, 1 << 20)
    out = ctx.malloc(0, 1 << 20)

    def outcome(fn):
        try:
            return {"ok": fn()}
        except rs.ReshardError as e:
            return {"error": e.name}

    for c in kat["slice"]:
        pay = np.frombuffer(bytes.fromhex(c["payload"]), np.uint8).copy()
        ctx.htod(0, buf, pay.ctypes.data, max(pay.size, 1))
        n = int(np.prod([z - a for a, z in c["box"]])) * W[c["dtype"]] if "ok" in c else 0

        def run():
            rs.slice(ctx, 0, rs.DeviceTensor(c["dtype"], tuple(c["shape"]), buf), [tuple(b) for b in c["box"]], out)
            got = np.zeros(n, np.uint8)
            ctx.dtoh(0, got.ctypes.data, out, n)
            return got.tobytes().hex()

        assert outcome(run) == {k: c[k] for k in ("ok", "error") if k in c}, c["shape"]
    for c in kat["merge"]:
        off, parts = 0, []
        for p in c["parts"]:
            pay = np.frombuffer(bytes.fromhex(p["payload"]), np.uint8).copy()
            if pay.size:
                ctx.htod(0, buf + off, pay.ctypes.data, pay.size)
            parts.append(([tuple(b) for b in p["box"]], rs.DeviceTensor(p["dtype"], tuple(p["shape"]), buf + off)))
            off += (pay.size + 255) // 256 * 256
        n = len(bytes.fromhex(c["ok"])) if "ok" in c else 0

        def run():
            rs.merge(ctx, 0, parts, tuple(c["target"]), out)
            got = np.zeros(n, np.uint8)
            ctx.dtoh(0, got.ctypes.data, out, n)
            return got.tobytes().hex()

        assert outcome(run) == {k: c[k] for k in ("ok", "error") if k in c}, c["target"]
    ctx.free(0, buf)
    ctx.free(0, out)


def test_identity_transition_moves_nothing(rs, orc, ctx):
    """(T,P,D) -> same (T,P,D): an empty plan; every destination cell is the kept source cell."""
    cat = rs.Catalog.gpt(64, 2, 16, 128, rs.MIXED_ADAM)
    a = cat.build_strategy(DEV(4), 2, 2, 1)
    plan = rs.generate_plan(a, cat.build_strategy(DEV(4), 2, 2, 1))
    assert plan.stats()["n_move"] == 0 and plan.stats()["moved_bytes"] == 0
    ex, t = _run(rs, ctx, plan, 4, 4)
    assert t[0]["bytes"] == 0
    assert ex.verify() == 0


def test_central_mode_same_final_state(rs, orc, ctx):
    """apply_plan(plan, central): every moved fragment staged on the
    central GPU, then re-uploaded — the destination cells equal the oracle's (and therefore
    distributed mode's) byte for byte; the executed bytes are 2 x moved + relayout."""
    entries = [("param/w", 0, (12, 8), 0, 0), ("param/v", 1, (6, 8), 1, 1), ("exp_avg/w", 0, (12, 8), 0, 0),
               ("param/b", 3, (5,), -1, -1)]
    for a_cfg, b_cfg, failed in [((2, 1, 1, DEV(2)), (1, 2, 1, DEV(2)), ()),
                                 ((2, 1, 1, DEV(2)), (2, 1, 2, DEV(4)), ()),
                                 ((2, 2, 1, DEV(4)), (4, 1, 1, DEV(4)), ()),
                                 ((2, 1, 2, DEV(4)), (2, 1, 1, [(0, 0), (0, 1)]), [(0, 2), (0, 3)])]:
        a, b, plan, oa, ob, oplan = _pair(rs, orc, entries, a_cfg, b_cfg, failed)
        n_src, n_dst = len(a_cfg[3]), len(b_cfg[3])
        ex = rs.Executor(ctx, plan, [0] * n_src, [0] * n_dst, 4096, central=0)
        ex.allocate_local()
        ex.prepare()
        ex.fill_sources()
        t = ex.apply()
        st = plan.stats()
        assert t[0]["bytes"] == 2 * st["moved_bytes"] + st["relayout_bytes"]
        assert ex.verify() == 0
        ostate = oplan.apply(oa.fill())[0]
        assert _compare_with_oracle(rs, ctx, ex, b, ostate, [d for d in b_cfg[3]]) > 0


@pytest.mark.parametrize("world,bulk_peer", [(4, "0"), (8, "0"), (8, "1")])
def test_single_process_multi_gpu_world_on_one_device(rs, orc, world, bulk_peer, monkeypatch):
    """One process driving a `world`-GPU world whose GPUs all map to cuda:0 (per-GPU streams,
    arenas and launches): logical device d runs on world GPU d % world, so most fragments
    have a destination on another world GPU (LDG/STG peer tiles beside the bulk kernel on
    a second stream, fan-out tiles with mixed local / remote replicas).  Every destination
    cell equals the oracle's.  RESHARD_BULK_PEER=1: TMA bulk stores to the other GPUs too."""
    monkeypatch.setenv("RESHARD_BULK_PEER", bulk_peer)
    ctx = rs.Context(world, list(range(world)), [0] * world)
    entries = [("param/w", 1, (16, 8), 0, 0), ("param/d", 1, (8, 16), 1, 0), ("exp_avg/w", 2, (16, 8), 0, 1),
               ("param/b", 3, (24,), 0, 1), ("param/ln", 2, (8,), -1, -1)]
    for a_cfg, b_cfg in [((2, 1, 1, DEV(2)), (2, 1, 2, DEV(4))),
                         ((4, 2, 1, DEV(8)), (2, 2, 2, DEV(8))),
                         ((2, 2, 2, DEV(8)), (4, 1, 1, DEV(4))),
                         ((1, 2, 1, DEV(2)), (2, 1, 4, DEV(8)))]:
        a, b, plan, oa, ob, oplan = _pair(rs, orc, entries, a_cfg, b_cfg)
        n_src, n_dst = len(a_cfg[3]), len(b_cfg[3])
        ex = rs.Executor(ctx, plan, [d % world for d in range(n_src)], [d % world for d in range(n_dst)], 4096)
        ex.allocate_local()
        ex.prepare()
        ex.fill_sources()
        t = ex.apply()
        assert len(t) == world
        assert ex.verify() == 0
        ostate = oplan.apply(oa.fill())[0]
        assert _compare_with_oracle(rs, ctx, ex, b, ostate, list(b_cfg[3])) > 0
        del ex


def test_reference_fixtures_through_host_value_api(rs, ctx):
    """The reference fixtures replayed through rs_slice_host / rs_merge_host (host buffers in
    and out, bytes moved on the GPU): same bytes, same error names."""
    kat = _kat()

    def outcome(fn):
        try:
            return {"ok": fn().hex()}
        except rs.ReshardError as e:
            return {"error": e.name}

    for c in kat["slice"]:
        got = outcome(lambda: rs.slice_host(ctx, 0, c["dtype"], c["shape"], bytes.fromhex(c["payload"]),
                                            [tuple(b) for b in c["box"]]))
        assert got == {k: c[k] for k in ("ok", "error") if k in c}, c["shape"]
    for c in kat["merge"]:
        parts = [([tuple(b) for b in p["box"]], p["dtype"], p["shape"], bytes.fromhex(p["payload"])) for p in c["parts"]]
        got = outcome(lambda: rs.merge_host(ctx, 0, parts, tuple(c["target"])))
        assert got == {k: c[k] for k in ("ok", "error") if k in c}, c["target"]


@pytest.mark.parametrize("kernel", ["bulk_strided", "bulk", "ldg", "bulk_dyn"])
def test_broadcast_fan_out_push(rs, ctx, kernel, monkeypatch):
    """rs_broadcast: one source to 1, 4, 6 destinations (fan-out groups of 4), aligned (TMA
    fan-out tiles) and misaligned (LDG/STG), every destination byte equal to the source."""
    monkeypatch.setenv("RESHARD_COPY_KERNEL", kernel)
    rng = np.random.default_rng(3)
    for nbytes, n_dst, skew in [(10 << 20, 6, 0), (1 << 20, 1, 0), (3 * 29696 + 48, 4, 0), (3 * 32768 + 48, 4, 0), (777_777, 3, 8), (96, 5, 0)]:
        src_h = rng.integers(0, 256, nbytes, dtype=np.uint8)
        src = ctx.malloc(0, nbytes + 64)
        ctx.htod(0, src + skew, src_h.ctypes.data, nbytes)
        dsts = [ctx.malloc(0, nbytes + 64) for _ in range(n_dst)]
        t = rs.broadcast(ctx, 0, src + skew, [d + skew for d in dsts], nbytes)
        assert t["bytes"] == nbytes * n_dst and t["launches"] == 1
        for d in dsts:
            got = np.empty(nbytes, np.uint8)
            ctx.dtoh(0, got.ctypes.data, d + skew, nbytes)
            assert np.array_equal(got, src_h)
            ctx.free(0, d)
        ctx.free(0, src)
    with pytest.raises(rs.ReshardError, match="InvalidArgument"):
        rs.broadcast(ctx, 0, 0, [1 << 20], 16)


def test_cell_larger_than_4gib(rs, ctx):
    """A single contiguous run above 2^32 bytes (one 4.5 GiB cell replicated to a new DP
    rank): the piece's run is 64-bit, its tiles are not; every destination byte verified."""
    n = (4 << 30) // 4 + (128 << 20)  # F32 elements: 4.5 GiB
    cat = rs.Catalog.from_entries([("param/huge", 0, (n,), -1, 0)])
    a = cat.build_strategy(DEV(1), 1, 1, 1)
    b = cat.build_strategy(DEV(2), 1, 1, 2)
    plan = rs.generate_plan(a, b)
    ex, t = _run(rs, ctx, plan, 1, 2)
    assert t[0]["bytes"] == 4 * n
    assert ex.verify() == 0


def test_tma_tensor_path_bytes_exact(rs, orc, ctx, monkeypatch):
    """K3T (RESHARD_TMA_TENSOR=1): strided row-mode pieces move as 3-D TMA tensor boxes
    (cp.async.bulk.tensor, one instruction per box; UTMALDG/UTMASTG in SASS) — random
    transitions with strided TP fragments, tile sizes that force partial boxes at the edges,
    and BASELINE configs[0] (dim-1 TP merges of 1536-byte rows), every destination byte
    equal to the oracle's."""
    monkeypatch.setenv("RESHARD_TMA_TENSOR", "1")
    rng = random.Random(99)
    ents = [("param/w", 0, (48, 40), 1, 0), ("param/v", 1, (64, 96), 1, 0), ("exp_avg/w", 2, (24, 16), 0, 1),
            ("param/big", 0, (40, 1152), 1, 1), ("param/ln", 0, (64,), -1, -1)]
    for (T1, P1, D1), (T2, P2, D2) in [((2, 1, 1), (1, 2, 1)), ((4, 2, 1), (2, 2, 2)), ((1, 1, 1), (4, 1, 2)),
                                       ((2, 2, 2), (4, 1, 1)), ((4, 1, 1), (2, 1, 1))]:
        n1, n2 = T1 * P1 * D1, T2 * P2 * D2
        a, b, plan, oa, ob, oplan = _pair(rs, orc, ents, (T1, P1, D1, DEV(n1)), (T2, P2, D2, DEV(n2)))
        for tile in (4096, 65536, 256 << 10):
            ex, _ = _run(rs, ctx, plan, n1, n2, tile)
            ost, _ = oplan.apply(oa.fill(), n_threads=4)
            _compare_with_oracle(rs, ctx, ex, b, ost, DEV(n2))
            assert ex.verify() == 0
            del ex
    cat = rs.Catalog.gpt(768, 12, 1024, 50304, rs.FP32_ADAM)
    a, b = cat.build_strategy(DEV(2), 2, 1, 1), cat.build_strategy(DEV(2), 1, 2, 1)
    ex, t = _run(rs, ctx, rs.generate_plan(a, b), 2, 2)
    assert ex.verify() == 0
    assert rng is not None


def test_execution_report_digests(rs, orc, ctx):
    """ExecutionReport verification digests: per base tensor, FNV-1a-64 of
    the tensor reassembled from the destination cells (one replica each) equals the digest
    reassembled from the source cells and the oracle's digest of the generated base tensor
    (End-to-end preservation) — for a reshard with splits, merges and DP
    replicas, and for the Fig. 6 transition."""
    cat = rs.Catalog.gpt(64, 4, 16, 128, rs.MIXED_ADAM)
    ocat = orc.catalog_gpt(64, 4, 16, 128, 1)
    for (T1, P1, D1), (T2, P2, D2) in [((4, 2, 1), (2, 2, 2)), ((2, 2, 2), (1, 4, 1)), ((1, 1, 1), (2, 1, 2))]:
        n1, n2 = T1 * P1 * D1, T2 * P2 * D2
        a, b = cat.build_strategy(DEV(n1), T1, P1, D1), cat.build_strategy(DEV(n2), T2, P2, D2)
        ex, _ = _run(rs, ctx, rs.generate_plan(a, b), n1, n2)
        src, dst = ex.digests(0), ex.digests(1)
        assert len(dst) == len(cat) and src == dst
        assert ex.digests(1, replica=-1) == dst  # the other DP copy of every replicated cell
        for t in range(0, len(cat), 7):
            assert dst[t] == ocat.base_digest(t), f"tensor {t}"
        del ex
    entries = [("t1", 0, (6,), 0, 0), ("t2", 0, (6,), 0, 1)]
    a, b, plan, oa, ob, oplan = _pair(rs, orc, entries, (2, 1, 1, DEV(2)), (3, 2, 1, DEV(6)))
    ex, _ = _run(rs, ctx, plan, 2, 6)
    ocat2 = orc.catalog(entries)
    assert ex.digests(1) == {0: ocat2.base_digest(0), 1: ocat2.base_digest(1)} == ex.digests(0)


@pytest.mark.parametrize("pipeline", ["1", "0"])
def test_run_host_world_matches_device_result(rs, pipeline, monkeypatch):
    """e2e through rs_executor_run_host_world over a 4- and an 8-GPU world in one process (all
    world GPUs on cuda:0): pipelined rounds (default) and the three-phase form.  Every source
    byte comes from the host buffers (device src arenas zeroed first), every destination cell
    verifies, and every GPU's host dst buffer equals its device dst arena (prefixes moved down
    while later rounds still push into the same arena included)."""
    monkeypatch.setenv("RESHARD_WORLD_PIPELINE", pipeline)
    cat = rs.Catalog.gpt(256, 6, 64, 1024, rs.MIXED_ADAM)
    for world, (a_cfg, b_cfg) in [(4, ((2, 1, 1, 2), (2, 1, 2, 4))), (8, ((4, 2, 1, 8), (2, 2, 2, 8))),
                                  (4, ((2, 2, 2, 8), (4, 1, 1, 4)))]:
        ctx = rs.Context(world, list(range(world)), [0] * world)
        a = cat.build_strategy(DEV(a_cfg[3]), *a_cfg[:3])
        b = cat.build_strategy(DEV(b_cfg[3]), *b_cfg[:3])
        ex = rs.Executor(ctx, rs.generate_plan(a, b), [d % world for d in range(a_cfg[3])],
                         [d % world for d in range(b_cfg[3])], 16 << 10)
        ex.allocate_local()
        ex.prepare()
        ex.fill_sources()
        hs, hd, sz = [0] * world, [0] * world, {}
        for g in range(world):
            s_b, d_b = ex.arena_bytes(g)
            sz[g] = (s_b, d_b)
            hs[g], hd[g] = rs.host_alloc(max(s_b, 1)), rs.host_alloc(max(d_b, 1))
            sp, dp = ex.arenas[g]
            ctx.dtoh(g, hs[g], sp, s_b)
            ctx.memset(g, sp, 0, s_b)
            ctx.memset(g, dp, 0, d_b)
        ms = ex.run_host_world(hs, hd)
        assert ms > 0
        assert ex.verify() == 0
        for g in range(world):
            d_b = sz[g][1]
            if not d_b:
                continue
            dev = np.zeros(d_b, np.uint8)
            ctx.dtoh(g, dev.ctypes.data, ex.arenas[g][1], d_b)
            host = np.ctypeslib.as_array((ctypes.c_uint8 * d_b).from_address(hd[g]))
            assert np.array_equal(dev, host), f"world {world} GPU {g}"
        for g in range(world):
            rs.host_free(hs[g])
            rs.host_free(hd[g])
        del ex


@pytest.mark.parametrize("tail", ["-1", "1", "4"])
def test_bulk_dyn_kernel_bytes_exact(rs, orc, ctx, monkeypatch, tail):
    """RESHARD_COPY_KERNEL=bulk_dyn (dynamic tile claims from a global counter that the last
    CTA resets): random transitions and repeated launches on one executor (the counter must be
    back at zero for every launch), every destination byte equal to the oracle's."""
    monkeypatch.setenv("RESHARD_COPY_KERNEL", "bulk_dyn")
    monkeypatch.setenv("RESHARD_DYN_TAIL", tail)  # dynamic claims for everything / the last 1 or 4 tiles per CTA
    cat = rs.Catalog.gpt(256, 6, 64, 1024, rs.MIXED_ADAM)
    for (a_cfg, b_cfg) in [((2, 1, 1, 2), (2, 1, 2, 4)), ((4, 2, 1, 8), (2, 2, 2, 8)), ((2, 1, 1, 2), (1, 2, 1, 2))]:
        a = cat.build_strategy(DEV(a_cfg[3]), *a_cfg[:3])
        b = cat.build_strategy(DEV(b_cfg[3]), *b_cfg[:3])
        ex, _ = _run(rs, ctx, rs.generate_plan(a, b), a_cfg[3], b_cfg[3], 16 << 10)
        for _ in range(3):
            ex.apply()
        assert ex.verify() == 0
        del ex


@pytest.mark.parametrize("world", [1, 4])
def test_ldg_dynamic_claims_bytes_exact(rs, orc, world, monkeypatch):
    """RESHARD_LDG_DYN=1: the LDG/STG kernels (K1 aligned, K2 fan-out incl. peer stores in a
    4-GPU world on cuda:0) claim tiles dynamically; repeated launches reuse the counter the last
    CTA resets; every destination cell equals the oracle's."""
    monkeypatch.setenv("RESHARD_LDG_DYN", "1")
    monkeypatch.setenv("RESHARD_COPY_KERNEL", "ldg" if world == 1 else "bulk_strided")
    ctx = rs.Context(world, list(range(world)), [0] * world)
    entries = [("param/w", 1, (64, 32), 0, 0), ("param/d", 1, (32, 64), 1, 0), ("exp_avg/w", 2, (64, 32), 0, 1),
               ("param/b", 3, (96,), 0, 1), ("param/ln", 2, (32,), -1, -1)]
    for a_cfg, b_cfg in [((2, 1, 1, DEV(2)), (2, 1, 2, DEV(4))), ((4, 2, 1, DEV(8)), (2, 2, 2, DEV(8))),
                         ((1, 2, 1, DEV(2)), (2, 1, 4, DEV(8)))]:
        a, b, plan, oa, ob, oplan = _pair(rs, orc, entries, a_cfg, b_cfg)
        n_src, n_dst = len(a_cfg[3]), len(b_cfg[3])
        ex = rs.Executor(ctx, plan, [d % world for d in range(n_src)], [d % world for d in range(n_dst)], 4096)
        ex.allocate_local()
        ex.prepare()
        ex.fill_sources()
        for _ in range(3):
            ex.apply()
        assert ex.verify() == 0
        ostate = oplan.apply(oa.fill())[0]
        assert _compare_with_oracle(rs, ctx, ex, b, ostate, list(b_cfg[3])) > 0
        del ex
