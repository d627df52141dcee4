"""The C-ABI library (CPU side): loads, exports every symbol include/reshard_b200.h declares,
and its host box algebra reproduces the reference tensor-core fixtures
(tests/golden/tensor_core_kat.json, generated from /root/reference/proj/src/tensor/*.cpp)."""
import ctypes
import json
import os
import re

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
KAT = json.load(open(os.path.join(HERE, "golden", "tensor_core_kat.json")))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "reshard_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rs_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(rs):
    syms = header_symbols()
    assert len(syms) > 50
    cdll = ctypes.CDLL(rs._capi.LIB_PATH)
    missing = [s for s in syms if not hasattr(cdll, s)]
    assert missing == []
    # and the Python binding declares a signature for each of them
    assert sorted(rs._capi.SIGNATURES) == syms


def test_sm100a_cubin_present(rs):
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", rs._capi.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_errc_numbering_matches_reference(rs):
    # error.hpp:8-48 order, then the appended device codes
    names = [rs.lib.rs_errc_name(i).decode() for i in range(rs.lib.rs_errc_count())]
    assert names[:32] == rs._capi.ERRC[:32]
    assert names[28] == "CheckpointRequired" and names[31] == "ScriptError"
    assert names[32:] == ["CudaError", "DeviceUnavailable", "InvalidArgument"]


def outcome(fn):
    try:
        return {"ok": fn()}
    except Exception as e:  # ReshardError
        return {"error": getattr(e, "name", type(e).__name__)}


def test_range_parse_fixtures(rs):
    for c in KAT["parse"]:
        if c["spec"]:
            continue
        got = outcome(lambda: [list(x) for x in rs.range_parse(c["text"])])
        assert got == {k: c[k] for k in ("ok", "error") if k in c}, c["text"]


def test_range_format_round_trip(rs):
    for c in KAT["parse"]:
        if "ok" in c and not c["spec"]:
            assert rs.range_format(c["ok"]) == c["text"]


def test_grid_fixtures(rs):
    for c in KAT["grid_cells"]:
        got = outcome(lambda: [[list(i) for i in cell] for cell in rs.grid_cells(tuple(c["shape"]), c["points"])])
        assert got == {k: c[k] for k in ("ok", "error") if k in c}, c
    for c in KAT["grid_refine"]:
        assert outcome(lambda: rs.grid_refine(c["a"], c["b"])) == {k: c[k] for k in ("ok", "error") if k in c}
    for c in KAT["even_split"]:
        got = outcome(lambda: rs.even_split(tuple(c["shape"]), c["dim"], c["ways"]))
        assert got == {k: c[k] for k in ("ok", "error") if k in c}, c


def _want(c):
    return {k: c[k] for k in ("ok", "error") if k in c}


def _lists(box):
    return [list(x) for x in box]


def test_cell_offset_resolve_fixtures(rs):
    """SplitGrid::cell / cell_index_of, Range::offset_by, RangeSpec resolve vs the reference."""
    for c in KAT["grid_cell"]:
        assert outcome(lambda: _lists(rs.grid_cell(tuple(c["shape"]), c["points"], c["index"]))) == _want(c), c
    for c in KAT["cell_index_of"]:
        assert outcome(lambda: rs.grid_cell_index_of(tuple(c["shape"]), c["points"], c["box"])) == _want(c), c
    for c in KAT["offset_by"]:
        assert outcome(lambda: _lists(rs.range_offset_by(c["box"], c["outer"]))) == _want(c), c
    for c in KAT["spec_resolve"]:
        assert outcome(lambda: _lists(rs.rangespec_resolve(c["text"], tuple(c["shape"])))) == _want(c), c
    for c in KAT["grid_cells"]:  # cell(i) enumerates cells() in order
        if "ok" in c:
            assert [_lists(rs.grid_cell(tuple(c["shape"]), c["points"], i)) for i in range(len(c["ok"]))] == c["ok"]
            for i, cell in enumerate(c["ok"]):
                assert rs.grid_cell_index_of(tuple(c["shape"]), c["points"], cell) == i


def test_valid_for_and_dtype_names(rs):
    assert rs.range_valid_for([(0, 4), (2, 4)], (4, 6))
    assert not rs.range_valid_for([(0, 4), (2, 7)], (4, 6))
    assert not rs.range_valid_for([(2, 2)], (4,))
    assert not rs.range_valid_for([(0, 1)], (4, 6))
    for name, code in [("f32", 0), ("F32", 0), ("f16", 1), ("i64", 2), ("U8", 3), ("bf16", 4), ("BF16", 4)]:
        assert rs.dtype_from_name(name) == code
    with pytest.raises(rs.ReshardError) as e:
        rs.dtype_from_name("fp8")
    assert e.value.name == "MalformedConfig"


def test_fnv_and_seed(rs, orc):
    assert rs.fnv1a64(b"") == 0xCBF29CE484222325
    for s in [b"a", b"param/embedding.word_embeddings.weight", bytes(range(200))]:
        assert rs.fnv1a64(s) == orc.fnv1a64(s)
    assert rs.payload_seed("param/x") == orc.path_seed("param/x")


def test_device_calls_fail_loudly_without_gpu(rs):
    if rs.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(rs.ReshardError) as e:
        rs.Context(1, [0], [0])
    assert e.value.name == "DeviceUnavailable"


def test_planning_only_context_lowers_tiles(rs):
    """A context with no local GPU computes arenas and tiles (used by the multi-rank
    bench to agree on layouts); it launches nothing."""
    cat = rs.Catalog.gpt(64, 2, 16, 128, rs.FP32_ADAM)
    a = cat.build_strategy([(0, 0), (0, 1)], 2, 1, 1)
    b = cat.build_strategy([(0, 0), (0, 1)], 1, 2, 1)
    plan = rs.generate_plan(a, b)
    ctx = rs.Context(2, [], [])
    ex = rs.Executor(ctx, plan, [0, 1], [0, 1], 4096)
    st = plan.stats()
    s0, d0 = ex.arena_bytes(0)
    s1, d1 = ex.arena_bytes(1)
    assert s0 + s1 >= cat.nbytes() and d0 + d1 >= st["dst_bytes"] - st["kept_bytes"]
    t0, b0 = ex.tiles(0)
    t1, b1 = ex.tiles(1)
    assert b0 + b1 == st["moved_bytes"] + st["relayout_bytes"]
    assert t0 > 0 and t1 > 0


def test_central_mode_layout_and_traffic(rs):
    """apply_plan(central): the central GPU stages every Move once, so its
    executed bytes are 2 x moved bytes (fetch + re-upload) plus local relayouts, its dst arena
    grows by the staging region, and the per-GPU traffic matches plan_cost_central."""
    cat = rs.Catalog.gpt(64, 4, 16, 128, rs.MIXED_ADAM)
    for (a_cfg, b_cfg) in [((2, 1, 1, 2), (1, 2, 1, 2)), ((2, 1, 1, 2), (2, 1, 2, 4)), ((4, 2, 1, 8), (2, 2, 2, 8))]:
        a = cat.build_strategy([(0, i) for i in range(a_cfg[3])], *a_cfg[:3])
        b = cat.build_strategy([(0, i) for i in range(b_cfg[3])], *b_cfg[:3])
        plan = rs.generate_plan(a, b)
        st = plan.stats()
        G = max(a_cfg[3], b_cfg[3])
        ctx = rs.Context(G, [], [])
        dist = rs.Executor(ctx, plan, list(range(a_cfg[3])), list(range(b_cfg[3])), 4096)
        cen = rs.Executor(ctx, plan, list(range(a_cfg[3])), list(range(b_cfg[3])), 4096, central=0)
        assert cen.staging_bytes() >= st["moved_bytes"]
        assert dist.staging_bytes() == 0
        assert cen.arena_bytes(0)[1] == dist.arena_bytes(0)[1] + cen.staging_bytes()
        total = sum(cen.tiles(g)[1] for g in range(G))
        assert total == 2 * st["moved_bytes"] + st["relayout_bytes"]
        # central GPU 0 re-uploads every moved byte; the others only fetch theirs
        fetch = sum(dist.tiles(g)[1] for g in range(G)) - st["relayout_bytes"]
        assert fetch == st["moved_bytes"]
        assert cen.tiles(0)[1] >= st["moved_bytes"]
    with pytest.raises(rs.ReshardError) as e:
        rs.Executor(rs.Context(2, [], []), plan, list(range(8)), list(range(8)), 4096, central=8)
    assert e.value.name == "InvalidArgument"


def test_dataset_abi_argument_errors(rs):
    """The dataset entry points validate their arguments before touching a device: null
    pointers and an unknown index layout fail with InvalidArgument (no exception crosses
    the C ABI; the message carries the Errc name like reshard::Error::what())."""
    import ctypes as C

    from paper_2312_05181_b200 import _capi

    lib = rs.lib
    ctx = rs.Context(1, [], [])
    t = _capi.rs_timing()
    inv = 1 + rs._capi.ERRC.index("InvalidArgument")
    assert lib.rs_dataset_index_upload(ctx.h, 0, None, None, 10, None, None, None, C.byref(t)) == inv
    assert "InvalidArgument" in lib.rs_last_error().decode()
    assert lib.rs_dataset_index_pad(ctx.h, 0, None, None, 10, C.byref(t)) == inv
    idx = _capi.rs_dataset_index(8, 8, 8, 100, 24)
    out = _capi.rs_partition_out()
    assert lib.rs_repartition_to_host(ctx.h, 0, C.byref(idx), 10, 0, 2, 0, C.byref(out), None, None, C.byref(t)) == inv
    host = _capi.rs_partition_host()
    out.pos = out.ent = out.boff = out.qcount = 8
    assert lib.rs_repartition_to_host(ctx.h, 0, C.byref(idx), 10, 0, 2, 0, C.byref(out), 8, C.byref(host),
                                      C.byref(t)) == inv  # null host buffers
    bad = _capi.rs_dataset_index(8, 8, 8, 100, 16)
    assert lib.rs_repartition(ctx.h, 0, C.byref(bad), 10, 0, 2, 0, C.byref(out), 8, C.byref(t)) == inv
    assert "entry_bytes" in lib.rs_last_error().decode()
    # rs_repartition_batch: null total / index, negative count, null job list, a job without
    # scratch or locator classes, a bad layout, then the SPEC's own errors — all before any device work
    jobs = (_capi.rs_repartition_job * 2)()
    for j in jobs:
        j.at_step, j.new_dp, j.rank, j.file_class, j.out, j.scratch = 0, 2, 0, 8, out, 8
    assert lib.rs_repartition_batch(ctx.h, 0, C.byref(idx), 10, jobs, 2, None, None) == inv
    assert lib.rs_repartition_batch(ctx.h, 0, None, 10, jobs, 2, None, C.byref(t)) == inv
    assert lib.rs_repartition_batch(ctx.h, 0, C.byref(idx), 10, jobs, -1, None, C.byref(t)) == inv
    assert "negative" in lib.rs_last_error().decode()
    assert lib.rs_repartition_batch(ctx.h, 0, C.byref(idx), 10, None, 2, None, C.byref(t)) == inv
    jobs[1].scratch = None
    assert lib.rs_repartition_batch(ctx.h, 0, C.byref(idx), 10, jobs, 2, None, C.byref(t)) == inv
    jobs[1].scratch, jobs[1].file_class = 8, None
    assert lib.rs_repartition_batch(ctx.h, 0, C.byref(idx), 10, jobs, 2, None, C.byref(t)) == inv
    jobs[1].file_class = 8
    assert lib.rs_repartition_batch(ctx.h, 0, C.byref(bad), 10, jobs, 2, None, C.byref(t)) == inv
    assert "entry_bytes" in lib.rs_last_error().decode()
    jobs[1].new_dp = 3  # B = 10 is not divisible by 3
    rc = lib.rs_repartition_batch(ctx.h, 0, C.byref(idx), 10, jobs, 2, None, C.byref(t))
    assert rc == 1 + rs._capi.ERRC.index("IndivisibleBatch"), lib.rs_last_error().decode()
    # run_host flags / upload bytes on a null executor
    b = C.c_uint64()
    assert lib.rs_executor_run_host_flags(None, 0, None, None, 1, C.byref(t)) == inv
    assert lib.rs_executor_host_upload_bytes(None, 0, 1, C.byref(b)) == inv


def _kat():
    import json

    return json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "tensor_core_kat.json")))


def test_host_value_slice_merge_validate_before_device(rs):
    """rs_slice_host / rs_merge_host (the reference's value-level slice / merge) check their
    arguments exactly like the reference before touching a device: every error case of the
    reference fixtures gives the reference's error name with no GPU present, and a valid call
    then fails with DeviceUnavailable (no CPU path)."""
    ctx = rs.Context(1, [], [])

    def outcome(fn):
        try:
            fn()
            return "ok"
        except rs.ReshardError as e:
            return e.name

    kat = _kat()
    for c in kat["slice"]:
        got = outcome(lambda: rs.slice_host(ctx, 0, c["dtype"], c["shape"], bytes.fromhex(c["payload"]),
                                            [tuple(b) for b in c["box"]]))
        assert got == (c["error"] if "error" in c else "DeviceUnavailable"), c
    for c in kat["merge"]:
        parts = [([tuple(b) for b in p["box"]], p["dtype"], p["shape"], bytes.fromhex(p["payload"])) for p in c["parts"]]
        got = outcome(lambda: rs.merge_host(ctx, 0, parts, tuple(c["target"])))
        assert got == (c["error"] if "error" in c else "DeviceUnavailable"), c


def test_broadcast_argument_errors(rs):
    """rs_broadcast rejects a null source / empty or null destination list before any device
    work (InvalidArgument)."""
    ctx = rs.Context(1, [], [])
    for src, dsts in [(0, [4096]), (4096, []), (4096, [0])]:
        with pytest.raises(rs.ReshardError) as e:
            rs.broadcast(ctx, 0, src, dsts, 64)
        assert e.value.name == "InvalidArgument"


def test_bytes_to_rows_of_the_all_to_all(rs):
    """Executor.bytes_to(g): GPU g's egress row of the fragment all-to-all.  Rows sum to the
    executed bytes, the DP scale-out 2 -> 4 over 4 GPUs moves the replicas across GPUs, and
    planning-only contexts (no GPU) compute it (the multi-rank bench's NVLink roofline)."""
    cat = rs.Catalog.gpt(64, 2, 16, 128, rs.MIXED_ADAM)
    a = cat.build_strategy([(0, 0), (0, 1)], 2, 1, 1)
    b = cat.build_strategy([(0, i) for i in range(4)], 2, 1, 2)
    plan = rs.generate_plan(a, b)
    ctx = rs.Context(4, [], [])
    ex = rs.Executor(ctx, plan, [0, 1], [0, 1, 2, 3], 4096)
    rows = [ex.bytes_to(g) for g in range(4)]
    for g in range(4):
        assert sum(rows[g]) == ex.tiles(g)[1]
    st = plan.stats()
    # every moved byte crosses to the new replica's GPUs (2, 3); choose_source balances the
    # egress of the two source GPUs
    assert sum(rows[0][2:]) + sum(rows[1][2:]) == st["moved_bytes"]
    assert abs(sum(rows[0]) - sum(rows[1])) < 0.1 * st["moved_bytes"]
    assert rows[0][:2] == [0, 0] and rows[1][:2] == [0, 0]  # the kept replica moves nothing
    assert rows[2] == [0, 0, 0, 0] and rows[3] == [0, 0, 0, 0]
