"""Pinning the CPU oracle (test infrastructure) before trusting it:
  * against the golden fixtures generated from the reference's own compiled tensor-core
    (tests/golden/make_golden.py; /root/reference/proj/src/tensor/*.cpp);
  * live against the reference build (oracle/_ref) on fresh random cases;
  * against the SPEC known-answer examples and the survey's derived KATs.
"""
import json
import os
import random

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
KAT = json.load(open(os.path.join(HERE, "golden", "tensor_core_kat.json")))
PLANS = json.load(open(os.path.join(HERE, "golden", "plans.json")))


def outcome(fn):
    from oracle.oracle import OracleError

    try:
        return {"ok": fn()}
    except OracleError as e:
        return {"error": e.name}


def norm(x):
    return json.loads(json.dumps(x))


@pytest.mark.parametrize("case", KAT["slice"], ids=lambda c: f"{c['shape']}{c['box']}")
def test_slice_matches_reference_fixture(orc, case):
    pay = np.frombuffer(bytes.fromhex(case["payload"]), np.uint8)
    got = outcome(lambda: orc.slice(case["dtype"], tuple(case["shape"]), pay,
                                    [tuple(b) for b in case["box"]]).tobytes().hex())
    assert got == {k: case[k] for k in ("ok", "error") if k in case}


def _parts(case):
    return [([tuple(b) for b in p["box"]], p["dtype"], tuple(p["shape"]), np.frombuffer(bytes.fromhex(p["payload"]), np.uint8))
            for p in case["parts"]]


def test_merge_matches_reference_fixture(orc):
    for case in KAT["merge"]:
        got = outcome(lambda: orc.merge(_parts(case), tuple(case["target"])).tobytes().hex())
        assert got == {k: case[k] for k in ("ok", "error") if k in case}, case["target"]


def test_grid_refine_split_parse_fixtures(orc):
    for c in KAT["grid_cells"]:
        got = outcome(lambda: orc.grid_cells(tuple(c["shape"]), c["points"]))
        assert norm(got) == {k: c[k] for k in ("ok", "error") if k in c}, c
    for c in KAT["grid_refine"]:
        assert norm(outcome(lambda: orc.grid_refine(c["a"], c["b"]))) == {k: c[k] for k in ("ok", "error") if k in c}
    for c in KAT["even_split"]:
        got = outcome(lambda: orc.even_split(tuple(c["shape"]), c["dim"], c["ways"]))
        assert norm(got) == {k: c[k] for k in ("ok", "error") if k in c}, c
    for c in KAT["parse"]:
        got = outcome(lambda: orc.range_parse(c["text"], c["spec"]))
        assert norm(got) == {k: c[k] for k in ("ok", "error") if k in c}, c


def _want(c):
    return {k: c[k] for k in ("ok", "error") if k in c}


def _tup(box):
    return [tuple(x) for x in box]


def test_cell_offset_resolve_fixtures(orc):
    for c in KAT["grid_cell"]:
        assert norm(outcome(lambda: orc.grid_cell(tuple(c["shape"]), c["points"], c["index"]))) == _want(c), c
    for c in KAT["cell_index_of"]:
        got = outcome(lambda: orc.grid_cell_index_of(tuple(c["shape"]), c["points"], _tup(c["box"])))
        assert got == _want(c), c
    for c in KAT["offset_by"]:
        assert norm(outcome(lambda: orc.offset_by(_tup(c["box"]), _tup(c["outer"])))) == _want(c), c
    for c in KAT["spec_resolve"]:
        spec = orc.range_parse(c["text"], True)
        assert norm(outcome(lambda: orc.spec_resolve(spec, tuple(c["shape"])))) == _want(c), c


def test_spec_kats(orc):
    f = np.arange(24, dtype=np.float32).view(np.uint8)
    out = np.frombuffer(orc.slice(0, (4, 6), f, [(0, 4), (2, 4)]).tobytes(), np.float32)
    assert out.tolist() == [2, 3, 8, 9, 14, 15, 20, 21]
    six = np.arange(6, dtype=np.float32).view(np.uint8)
    assert np.frombuffer(orc.slice(0, (6,), six, [(2, 3)]).tobytes(), np.float32).tolist() == [2]
    assert orc.grid_refine([[3]], [[2, 4]]) == [[2, 3, 4]]
    assert orc.grid_cells((6,), [[2, 4]]) == [[(0, 2)], [(2, 4)], [(4, 6)]]
    assert orc.grid_cells((4, 6), [[], [3]]) == [[(0, 4), (0, 3)], [(0, 4), (3, 6)]]
    assert orc.fnv1a64(b"") == 0xCBF29CE484222325
    assert orc.splitmix64(0, 1)[0][0] == 0xE220A8397B1DCDAF
    v, st = orc.next_below(5, 0)
    assert v == 0 and st == 5                                                 # hash.hpp:59, no advance


def test_restatement_vs_reference_live(orc, ref):
    rng = random.Random(99)
    for _ in range(300):
        rank = rng.randint(0, 4)
        shape = tuple(rng.randint(1, 6) for _ in range(rank))
        dt = rng.choice([0, 1, 2, 3])
        pay = np.frombuffer(rng.randbytes(int(np.prod(shape)) * {0: 4, 1: 2, 2: 8, 3: 1}[dt]), np.uint8)
        box = [(a, rng.randint(a + 1, e + 1)) for e in shape for a in [rng.randint(0, e - 1)]]
        assert outcome(lambda: orc.slice(dt, shape, pay, box).tobytes()) == outcome(lambda: ref.slice(dt, shape, pay, box).tobytes())
        pts = [sorted(rng.sample(range(1, e), rng.randint(0, min(2, e - 1)))) if e > 1 else [] for e in shape]
        assert outcome(lambda: orc.grid_cells(shape, pts)) == outcome(lambda: ref.grid_cells(shape, pts))
        cells = ref.grid_cells(shape, pts)
        parts = [(c, dt, tuple(z - a for a, z in c), ref.slice(dt, shape, pay, c)) for c in cells]
        if parts and rng.random() < 0.3:
            parts = parts[1:] if rng.random() < 0.5 else parts + parts[:1]
        assert outcome(lambda: orc.merge(parts, shape).tobytes()) == outcome(lambda: ref.merge(parts, shape).tobytes())
    for s in range(50):
        st = rng.getrandbits(64)
        assert orc.splitmix64(st, 4) == ref.splitmix64(st, 4)
        n = rng.randint(0, 1000)
        assert orc.next_below(st, n) == ref.next_below(st, n)
        data = rng.randbytes(rng.randint(0, 64))
        assert orc.fnv1a64(data) == ref.fnv1a64(data)


def test_payload_stream_matches_slice_of_base(orc):
    """gen_box (counter-based stream of a sub-box) == slice(full base stream, box)."""
    cat = orc.catalog([("a/x", 0, (6, 10), 0, 0), ("b/y", 1, (7, 3, 5), 1, 0), ("c/z", 3, (13,), 0, 0),
                       ("d/w", 2, (3, 4), -1, 0)])
    rng = random.Random(3)
    for t, (_, dt, shape, _, _) in enumerate(cat.entries()):
        full = cat.base_bytes(t)
        seed = orc.path_seed(cat.entry(t)[0])
        assert np.array_equal(full, orc.stream_bytes(seed, 0, full.size))
        for _ in range(20):
            box = [(a, rng.randint(a + 1, e)) for e in shape for a in [rng.randint(0, e - 1)]]
            assert np.array_equal(cat.box_bytes(t, box), orc.slice(dt, shape, full, box))


def test_fig6_golden_plan(orc):
    """Acceptance #4: refinement [2,3,4], 4 splits, 6 moves / 36 bytes, one
    two-fragment merge per middle cell, no move of a destination-resident fragment."""
    cat = orc.catalog([("t1", 0, (6,), 0, 0), ("t2", 0, (6,), 0, 1)])
    a = cat.build_strategy([(0, 0), (0, 1)], 2, 1, 1)
    b = cat.build_strategy([(0, i) for i in range(6)], 3, 2, 1)
    p = a.plan(b)
    assert p.text() == open(os.path.join(HERE, "golden", "fig6_plan.txt")).read()
    st = p.stats()
    assert (st["n_split"], st["n_move"], st["n_merge"], st["moved_bytes"]) == (4, 6, 2, 36)
    assert st["relayout_bytes"] == 12  # resident non-moved: dev0 8 B + dev1 4 B
    src, _ = a.fill(), None
    dst, rep = p.apply(src, n_threads=6)
    assert rep["moved"] == 36 and rep["local"] == 12
    assert all(b.digest(dst, t) == cat.base_digest(t) for t in range(2))


@pytest.mark.parametrize("name", sorted(PLANS))
def test_baseline_plan_statistics(orc, name):
    import bench

    (h, L, S, V, k), (T1, P1, D1, d1), (T2, P2, D2, d2), failed = bench.WORKLOADS[name]
    cat = orc.catalog_gpt(h, L, S, V, k)
    p = cat.build_strategy([(0, d) for d in d1], T1, P1, D1).plan(cat.build_strategy([(0, d) for d in d2], T2, P2, D2),
                                                                 failed=[(0, d) for d in failed])
    want = PLANS[name]
    cost = p.cost()
    got = {**p.stats(), "max_ingress": max(v[0] for v in cost.values()), "max_egress": max(v[1] for v in cost.values()),
           "text_fnv1a64": orc.fnv1a64(p.text().encode())}
    assert got == want


def _rand_catalog(rng, n_t):
    ents = []
    for i in range(n_t):
        rank = rng.choice([1, 2, 2, 3])
        shape = tuple(rng.choice([1, 2, 3, 4, 6, 8, 12, 24]) for _ in range(rank))
        ents.append((f"t{i}", rng.choice([0, 1, 2, 3]), shape, rng.choice([-1] + list(range(rank))), i))
    return ents


def test_acceptance1_end_to_end_preservation(orc):
    """SPEC acceptance #1 on the oracle itself: >=200 random transitions, reassembled base
    tensors bit-identical (catalog <= 6 tensors, extents <= 24, devices <= 8)."""
    rng = random.Random(5)
    cfgs = [(T, P, D) for T in (1, 2, 3, 4) for P in (1, 2, 3) for D in (1, 2, 4) if T * P * D <= 8]
    done = 0
    while done < 200:
        ents = _rand_catalog(rng, rng.randint(1, 6))
        (T1, P1, D1), (T2, P2, D2) = rng.choice(cfgs), rng.choice(cfgs)
        if max(P1, P2) > len(ents):
            continue
        if any(tp >= 0 and (sh[tp] % T1 or sh[tp] % T2) for _, _, sh, tp, _ in ents):
            continue
        cat = orc.catalog(ents)
        n1, n2 = T1 * P1 * D1, T2 * P2 * D2
        base = rng.choice([0, n1])
        a = cat.build_strategy([(0, i) for i in range(n1)], T1, P1, D1)
        b = cat.build_strategy([(0, base + i) for i in range(n2)], T2, P2, D2)
        p = a.plan(b)
        dst, _ = p.apply(a.fill(), n_threads=3)
        for t in range(len(ents)):
            assert b.digest(dst, t) == cat.base_digest(t)
        done += 1
