"""PTX1 codec (declared by the reference at ptx_io.hpp:10-20 without an
implementation) and checkpoints (acceptance #7's checkpoint path)."""
import os
import struct

import numpy as np
import pytest

DEV = lambda n, w=0: [(w, i) for i in range(n)]  # noqa: E731


def ptx_ref(dtype, shape, payload):
    """The format as SPEC.md:104 states it, restated independently of the library."""
    return b"PTX1" + struct.pack("<BB", dtype, len(shape)) + b"".join(struct.pack("<Q", e) for e in shape) + payload


def test_ptx_round_trip_and_format(rs):
    from paper_2312_05181_b200 import checkpoint as ck

    rng = np.random.default_rng(0)
    for dtype, w in [(0, 4), (1, 2), (2, 8), (3, 1)]:
        for shape in [(), (5,), (3, 4), (2, 3, 4)]:
            n = int(np.prod(shape)) if shape else 1
            pay = rng.integers(0, 256, n * w, dtype=np.uint8).tobytes()
            enc = ck.ptx_encode(dtype, shape, pay)
            assert enc == ptx_ref(dtype, shape, pay)
            assert ck.ptx_encoded_size(dtype, shape) == len(enc)
            assert ck.ptx_decode(enc) == (dtype, tuple(shape), pay)
    # BF16 is written with the F16 code so reference readers accept it
    assert ck.ptx_encode(rs.BF16, (2,), b"\0" * 4)[4] == 1


@pytest.mark.parametrize("bad", [b"", b"PTX", b"PTX2\x00\x01" + b"\0" * 8 + b"\0" * 4, b"PTX1\x04\x01" + struct.pack("<Q", 1) + b"\0",
                                 b"PTX1\x00\x01" + struct.pack("<Q", 2) + b"\0" * 4,
                                 b"PTX1\x00\x02" + struct.pack("<Q", 1),
                                 b"PTX1\x03\x01" + struct.pack("<Q", 0)])
def test_ptx_malformed(rs, bad):
    from paper_2312_05181_b200 import checkpoint as ck

    with pytest.raises(rs.ReshardError) as e:
        ck.ptx_decode(bad)
    assert e.value.name == "InvalidTensor"


@pytest.mark.gpu
def test_checkpoint_round_trip_and_recovery(rs, ctx, tmp_path):
    """save the (4,2,1) state -> load it into a fresh executor -> reshard -> every byte
    verifies; a wrong rank set is LayoutMismatch; and the CheckpointRequired path of
    acceptance #7: (T,P,D)=(2,2,1) loses a device, recover() refuses, the checkpoint of
    the old layout is loaded and resharded onto the survivors instead."""
    from paper_2312_05181_b200 import checkpoint as ck

    cat = rs.Catalog.gpt(64, 4, 16, 128, rs.MIXED_ADAM)
    a = cat.build_strategy(DEV(8), 4, 2, 1)
    b = cat.build_strategy(DEV(8), 2, 2, 2)
    plan = rs.generate_plan(a, b)
    ex = rs.Executor(ctx, plan, [0] * 8, [0] * 8)
    ex.allocate_local()
    ex.prepare()
    ex.fill_sources()
    d = str(tmp_path / "ckpt")
    st = ck.checkpoint_save(ex, d, side=0)
    assert st["files"] == sum(len(a.hosted_subtensors(x)) for x in DEV(8))
    assert sorted(os.listdir(d)) == sorted(str(i) for i in range(8))
    # fresh executor, zeroed arenas, load, run, verify
    ex2 = rs.Executor(ctx, plan, [0] * 8, [0] * 8)
    ex2.allocate_local()
    ex2.prepare()
    s_bytes, _ = ex2.arena_bytes(0)
    ctx.memset(0, ex2.arenas[0][0], 0, s_bytes)
    ld = ck.checkpoint_load(ex2, d)
    assert ld["bytes"] == st["bytes"]
    ex2.apply()
    assert ex2.verify() == 0
    # destination layout saved and reloaded as the source of the reverse plan
    d2 = str(tmp_path / "ckpt_b")
    ck.checkpoint_save(ex2, d2, side=1)
    back = rs.generate_plan(b, a)
    ex3 = rs.Executor(ctx, back, [0] * 8, [0] * 8)
    ex3.allocate_local()
    ex3.prepare()
    ck.checkpoint_load(ex3, d2)
    ex3.apply()
    assert ex3.verify() == 0
    # LayoutMismatch: a 4-device layout cannot load the 8-rank checkpoint
    small = rs.generate_plan(cat.build_strategy(DEV(4), 2, 2, 1), cat.build_strategy(DEV(4), 2, 2, 1))
    ex4 = rs.Executor(ctx, small, [0] * 4, [0] * 4)
    ex4.allocate_local()
    with pytest.raises(rs.ReshardError) as e:
        ck.checkpoint_load(ex4, d)
    assert e.value.name == "LayoutMismatch"
    # acceptance #7, checkpoint path: D=1, device 3 fails -> CheckpointRequired
    c = cat.build_strategy(DEV(4), 2, 2, 1)
    survivors = [(0, 0), (0, 1)]
    target = cat.build_strategy(survivors, 1, 2, 1)
    with pytest.raises(rs.ReshardError) as e:
        rs.recover(c, [(0, 3)], target)
    assert e.value.name == "CheckpointRequired"
    ex5 = rs.Executor(ctx, rs.generate_plan(c, c), [0] * 4, [0] * 4)
    ex5.allocate_local()
    ex5.prepare()
    ex5.fill_sources()
    d3 = str(tmp_path / "ckpt_c")
    ck.checkpoint_save(ex5, d3, side=0)
    rec = rs.generate_plan(c, target)  # checkpoint layout -> survivors
    ex6 = rs.Executor(ctx, rec, [0] * 4, [0] * 2)
    ex6.allocate_local()
    ex6.prepare()
    ck.checkpoint_load(ex6, d3)
    ex6.apply()
    assert ex6.verify() == 0


def test_checkpoint_rejects_escaping_tensor_paths(rs, tmp_path):
    """A tensor path that is absolute or climbs with '..' is refused before anything is
    written: checked on a planning-only context, no GPU needed."""
    from paper_2312_05181_b200 import checkpoint as ck

    for bad in ("/tmp/x", "a/../../x"):
        cat = rs.Catalog.from_entries([(bad, 0, (8,), 0, 0)])
        a = cat.build_strategy(DEV(2), 2, 1, 1)
        ctx = rs.Context(1, [], [])
        ex = rs.Executor(ctx, rs.generate_plan(a, a), [0, 0], [0, 0])
        with pytest.raises(rs.ReshardError) as e:
            ck.checkpoint_save(ex, str(tmp_path / "c"), side=0)
        assert e.value.name == "InvalidArgument"
        assert not os.path.exists(tmp_path / "c")


@pytest.mark.gpu
def test_checkpoint_rank_hosting_two_cells(rs, ctx, tmp_path):
    """A rank may host several cells of one tensor (parse_parallel_config accepts it): each
    cell gets its own file (<path>.c<cell>.ptx), and the round trip restores both."""
    import json

    from paper_2312_05181_b200 import checkpoint as ck
    from paper_2312_05181_b200.config import parse_parallel_config

    leaf = lambda r: {"base": "w", "shape": [12, 4], "range": r, "dtype": "f32"}  # noqa: E731
    doc = json.dumps([{"w0": leaf([[0, 3], [0, 4]]), "w1": leaf([[3, 6], [0, 4]])},
                      {"w2": leaf([[6, 12], [0, 4]])}])
    a = parse_parallel_config(doc)
    assert len(a.hosted_subtensors((0, 0))) == 2
    b = rs.Catalog.from_entries([("w", 0, (12, 4), 0, 0)]).build_strategy(DEV(2), 1, 1, 2)
    plan = rs.generate_plan(a, b)
    ex = rs.Executor(ctx, plan, [0, 0], [0, 0])
    ex.allocate_local()
    ex.prepare()
    ex.fill_sources()
    d = str(tmp_path / "two")
    st = ck.checkpoint_save(ex, d, side=0)
    assert st["files"] == 3
    assert sorted(os.listdir(os.path.join(d, "0"))) == ["w.c0.ptx", "w.c1.ptx"]
    assert os.listdir(os.path.join(d, "1")) == ["w.ptx"]
    ex2 = rs.Executor(ctx, plan, [0, 0], [0, 0])
    ex2.allocate_local()
    ex2.prepare()
    ctx.memset(0, ex2.arenas[0][0], 0, ex2.arena_bytes(0)[0])
    ck.checkpoint_load(ex2, d)
    ex2.apply()
    assert ex2.verify() == 0
