"""Planner / collection-description parity (CPU): the product's host C++ (through the C-ABI)
against the oracle, plus the SPEC examples of parallel-config and
planner and acceptance criteria #2, #3, #5, #7."""
import itertools
import json
import os
import random

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
PLANS = json.load(open(os.path.join(HERE, "golden", "plans.json")))
DEV = lambda n, base=0, w=0: [(w, base + i) for i in range(n)]  # noqa: E731


def both(rs, orc, ents):
    return rs.Catalog.from_entries(ents), orc.catalog(ents)


def rand_entries(rng, n_t, extents=(1, 2, 3, 4, 6, 8, 12, 24)):
    ents = []
    for i in range(n_t):
        rank = rng.choice([1, 2, 2, 3])
        shape = tuple(rng.choice(extents) for _ in range(rank))
        ents.append((f"m/t{i}", rng.choice([0, 1, 2, 3]), shape, rng.choice([-1] + list(range(rank))), i))
    return ents


CFGS = [(T, P, D) for T in (1, 2, 3, 4) for P in (1, 2, 3) for D in (1, 2, 4) if T * P * D <= 8]


def test_random_plans_identical_to_oracle(rs, orc):
    """>= 300 random transitions (fresh / overlapping device sets, multi-worker clusters):
    plan text, statistics and cost table byte-identical to the oracle."""
    rng = random.Random(11)
    done = 0
    while done < 300:
        ents = rand_entries(rng, rng.randint(1, 6))
        (T1, P1, D1), (T2, P2, D2) = rng.choice(CFGS), rng.choice(CFGS)
        if max(P1, P2) > len(ents) or any(tp >= 0 and (s[tp] % T1 or s[tp] % T2) for _, _, s, tp, _ in ents):
            continue
        n1, n2 = T1 * P1 * D1, T2 * P2 * D2
        workers = rng.choice([1, 2, 4])
        d1 = [(i % workers, i // workers) for i in range(n1)]
        d2 = [((i + rng.choice([0, 1])) % workers, i // workers + rng.choice([0, 0, 8])) for i in range(n2)]
        if len(set(d2)) != n2:
            continue
        cat, ocat = both(rs, orc, ents)
        a, b = cat.build_strategy(d1, T1, P1, D1), cat.build_strategy(d2, T2, P2, D2)
        oa, ob = ocat.build_strategy(d1, T1, P1, D1), ocat.build_strategy(d2, T2, P2, D2)
        p, op = rs.generate_plan(a, b), oa.plan(ob)
        assert p.text() == op.text()
        assert p.stats() == op.stats()
        assert p.cost() == op.cost()
        done += 1


@pytest.mark.parametrize("name", sorted(PLANS))
def test_baseline_configs_match_golden(rs, name):
    import bench

    cat, a, b, plan, _, _ = bench.build_plan(rs, name, 1)
    cost = plan.cost()
    got = {**plan.stats(), "max_ingress": max(v[0] for v in cost.values()),
           "max_egress": max(v[1] for v in cost.values()), "text_fnv1a64": rs.fnv1a64(plan.text().encode())}
    assert got == PLANS[name]


def test_catalog_matches_oracle(rs, orc):
    for kind in (0, 1, 2):
        c, o = rs.Catalog.gpt(768, 12, 1024, 50304, kind), orc.catalog_gpt(768, 12, 1024, 50304, kind)
        ce, oe = c.entries(), o.entries()
        assert len(ce) == len(oe) == 148 * (3, 4, 1)[kind]
        for x, y in zip(ce, oe):
            assert (x[0], x[2], x[3], x[4]) == (y[0], y[2], y[3], y[4])
            assert (x[1] if x[1] != rs.BF16 else 1) == y[1]  # bf16 carried as F16 in the oracle
    n_params = sum(1 for e in rs.Catalog.gpt(768, 12, 1024, 50304, 2).entries() for _ in [0])
    assert n_params == 148
    total = rs.Catalog.gpt(768, 12, 1024, 50304, 2).nbytes() // 4
    assert total == 124_475_904
    assert rs.Catalog.gpt(2048, 24, 2048, 50304, 2).nbytes() // 4 == 1_315_819_520
    assert rs.Catalog.gpt(4096, 32, 2048, 50304, 2).nbytes() // 4 == 6_658_596_864


def test_identity_plan_empty(rs):
    """Acceptance #2: generate_plan(p, p) is empty for every builder output."""
    cat = rs.Catalog.gpt(64, 4, 16, 128, rs.MIXED_ADAM)
    for T, P, D in [(1, 1, 1), (2, 1, 1), (1, 2, 1), (2, 2, 2), (4, 2, 1), (1, 4, 2)]:
        a = cat.build_strategy(DEV(T * P * D), T, P, D)
        p = rs.generate_plan(a, a)
        assert p.text() == ""
        st = p.stats()
        assert st["moved_bytes"] == 0 and st["n_move"] == st["n_split"] == st["n_merge"] == 0
        assert st["kept_bytes"] == st["dst_bytes"]
        assert all(v == (0, 0) for v in p.cost().values())


def test_fig6(rs):
    cat = rs.Catalog.from_entries([("t1", 0, (6,), 0, 0), ("t2", 0, (6,), 0, 1)])
    p = rs.generate_plan(cat.build_strategy(DEV(2), 2, 1, 1), cat.build_strategy(DEV(6), 3, 2, 1))
    assert p.text() == open(os.path.join(HERE, "golden", "fig6_plan.txt")).read()
    assert p.cost()[(0, 1)] == (4, 20)


def test_minimality_brute_force(rs):
    """Acceptance #3: on exhaustive tiny instances (1 tensor, extent <= 6, <= 4 devices) the
    moved bytes equal the lower bound sum over (destination, needed fragment) of the bytes
    of fragments absent from the destination."""
    for ext in range(1, 7):
        for (T1, P1, D1), (T2, P2, D2) in itertools.product([(t, 1, d) for t in (1, 2, 3, 6) for d in (1, 2, 4)
                                                              if t * d <= 4 and ext % t == 0], repeat=2):
            if ext % T2:
                continue
            for base in (0, 2):
                cat = rs.Catalog.from_entries([("x", 3, (ext,), 0, 0)])
                d1, d2 = DEV(T1 * D1), DEV(T2 * D2, base)
                a, b = cat.build_strategy(d1, T1, P1, D1), cat.build_strategy(d2, T2, P2, D2)
                p = rs.generate_plan(a, b)
                # lower bound from first principles (elements of the byte tensor)
                held = {}
                for dv in d1:
                    for _, box in a.hosted_subtensors(dv):
                        held.setdefault(dv, set()).update(range(box[0][0], box[0][1]))
                lb = 0
                for dv in d2:
                    for _, box in b.hosted_subtensors(dv):
                        lb += sum(1 for e in range(box[0][0], box[0][1]) if e not in held.get(dv, set()))
                assert p.stats()["moved_bytes"] == lb, (ext, T1, D1, T2, D2, base)


def test_redeployment_moves_only(rs):
    """Acceptance #5: (4,2,1) on 8 devices -> same config on 8 fresh devices: only Moves,
    moved bytes == hosted model bytes."""
    cat = rs.Catalog.gpt(64, 4, 16, 128, rs.MIXED_ADAM)
    a = cat.build_strategy(DEV(8), 4, 2, 1)
    b = cat.build_strategy(DEV(8, w=1), 4, 2, 1)
    p = rs.generate_plan(a, b)
    st = p.stats()
    assert st["n_split"] == st["n_merge"] == 0 and st["n_move"] > 0
    assert st["moved_bytes"] == st["dst_bytes"]
    assert all(line.startswith("MOVE") for line in p.text().splitlines())


def test_dp_scaleout_moves_full_partitions(rs):
    """pure DP 2->4: new devices receive full model tensors via Moves."""
    cat = rs.Catalog.gpt(64, 2, 16, 128, rs.FP32_ADAM)
    p = rs.generate_plan(cat.build_strategy(DEV(2), 1, 1, 2), cat.build_strategy(DEV(4), 1, 1, 4))
    st = p.stats()
    assert st["n_split"] == st["n_merge"] == 0
    assert st["moved_bytes"] == 2 * cat.nbytes()
    cost = p.cost()
    assert cost[(0, 2)][0] == cost[(0, 3)][0] == cat.nbytes()
    # greedy least-egress source choice: both replicas serve, imbalance below one tensor
    e0, e1 = cost[(0, 0)][1], cost[(0, 1)][1]
    largest = max(4 * __import__("math").prod(s) for _, _, s, _, _ in cat.entries())
    assert e0 + e1 == 2 * cat.nbytes() and abs(e0 - e1) <= largest


def test_recovery(rs):
    """Acceptance #7: (4,2,2) losing one replica recovers from the other
    with zero checkpoint reads; losing both replicas of a cell -> CheckpointRequired."""
    cat = rs.Catalog.gpt(64, 4, 16, 128, rs.MIXED_ADAM)
    a = cat.build_strategy(DEV(16), 4, 2, 2)
    survivors = DEV(8)
    b = cat.build_strategy(DEV(8, w=1), 4, 2, 1)  # replacement devices
    p = rs.recover(a, DEV(8, 8), b)
    st = p.stats()
    assert st["moved_bytes"] == st["dst_bytes"]
    for line in p.text().splitlines():
        src = line.split()[3]
        assert int(src.split(":")[1]) < 8  # every source survived
    with pytest.raises(rs.ReshardError) as e:
        rs.recover(a, [(0, 0), (0, 8)], b)  # both replicas of (pp0, tp0)
    assert e.value.name == "CheckpointRequired"
    d1 = cat.build_strategy(DEV(8), 4, 2, 1)
    with pytest.raises(rs.ReshardError) as e:
        rs.recover(d1, [(0, 3)], cat.build_strategy([(0, 0), (0, 1), (0, 2), (0, 4)], 2, 2, 1))
    assert e.value.name == "CheckpointRequired"      # D=1, any failure
    with pytest.raises(rs.ReshardError) as e:      # the target may not contain a failed device
        rs.recover(a, DEV(8, 8), cat.build_strategy(DEV(16), 4, 2, 2))
    assert e.value.name == "InvalidArgument"
    # a failed device that hosts only replicas others still hold moves nothing extra
    assert survivors


def test_build_strategy_examples_and_errors(rs):
    cat = rs.Catalog.from_entries([("a", 0, (4, 6), 1, 0), ("b", 0, (6,), 0, 1)])
    # Fig. 5 shape: T=2, P=1, D=2 on 4 devices: each device holds one column of each tensor
    p = cat.build_strategy(DEV(4), 2, 1, 2)
    assert p.hosted_subtensors((0, 0)) == [(0, [(0, 4), (0, 3)]), (1, [(0, 3)])]
    assert p.hosted_subtensors((0, 3)) == [(0, [(0, 4), (3, 6)]), (1, [(3, 6)])]
    assert p.validate() == []
    # T=1, P=1, D=k: everything full everywhere
    p = cat.build_strategy(DEV(3), 1, 1, 3)
    assert all(len(p.hosted_subtensors(d)) == 2 for d in DEV(3))
    # T=1, P=k: tensor i -> stage i
    p = cat.build_strategy(DEV(2), 1, 2, 1)
    assert p.hosted_subtensors((0, 0)) == [(0, [(0, 4), (0, 6)])]
    assert p.hosted_subtensors((0, 1)) == [(1, [(0, 6)])]

    def err(fn):
        with pytest.raises(rs.ReshardError) as e:
            fn()
        return e.value.name

    assert err(lambda: cat.build_strategy(DEV(3), 2, 1, 1)) == "DeviceCountMismatch"
    assert err(lambda: cat.build_strategy(DEV(4), 4, 1, 1)) == "IndivisibleSliceDim"
    assert err(lambda: cat.build_strategy(DEV(3), 1, 3, 1)) == "IndivisibleLayerCount"
    assert err(lambda: cat.build_strategy(DEV(0), 0, 1, 1)) == "InvalidJobConfig"
    assert err(lambda: p.hosted_subtensors((5, 5))) == "UnknownDevice"
    bad = rs.Catalog.from_entries([("a", 0, (4,), 2, 0)])
    assert err(lambda: bad.build_strategy(DEV(2), 2, 1, 1)) == "RankMismatch"


def test_stage_balancing_remainder_first(rs, orc):
    ents = [(f"l{i}", 0, (4,), -1, i) for i in range(7)]
    cat, ocat = both(rs, orc, ents)
    p = cat.build_strategy(DEV(3), 1, 3, 1)
    stages = [[t for t, _ in p.hosted_subtensors(d)] for d in DEV(3)]
    assert stages == [[0, 1, 2], [3, 4], [5, 6]]  # 7 layers -> 3,2,2
    op = ocat.build_strategy(DEV(3), 1, 3, 1)
    assert [[t for t, _ in op.hosted(d)] for d in DEV(3)] == stages


def test_validate_examples(rs, orc):
    cat = rs.Catalog.from_entries([("a", 0, (5,), -1, 0), ("b", 0, (6,), 0, 0)])
    p = cat.build_strategy(DEV(2), 2, 1, 1)
    assert p.validate() == []
    p.set_alpha(0, [])  # partition (stage 0, tp 0) mapped to zero devices
    v = p.validate()
    assert len(v) == 1 and v[0].startswith("UnhostedPartition")
    q = cat.build_strategy(DEV(2), 2, 1, 1)
    q.set_sigma(0, [[7]])  # split point 7 on extent 5
    v = q.validate()
    assert len(v) == 1 and v[0].startswith("InvalidSplitPoint")
    # expert parallelism: sigma identity, phi grouping experts -> valid
    ep = rs.Catalog.from_entries([(f"expert{i}.w", 0, (4, 4), -1, i) for i in range(4)]).build_strategy(DEV(4), 1, 4, 1)
    assert ep.validate() == []
    # sequence parallelism: sigma slicing a data tensor along the sequence dim
    sp = rs.Catalog.from_entries([("data.tokens", 2, (8, 1024), 1, 0)]).build_strategy(DEV(4), 4, 1, 1)
    assert sp.validate() == [] and sp.hosted_subtensors((0, 2)) == [(0, [(0, 8), (512, 768)])]


def test_choose_source_examples(rs):
    """SPEC.md:241-243."""
    assert rs.choose_source([(0, 0), (0, 1)], [5, 0], (0, 0)) == (0, 0)          # resident
    assert rs.choose_source([(0, 1), (1, 0)], [0, 0], (0, 0)) == (0, 1)          # same worker
    assert rs.choose_source([(1, 3), (1, 5)], [7, 7], (0, 0)) == (1, 3)          # tie -> smallest id
    assert rs.choose_source([(1, 3), (1, 5)], [9, 7], (0, 0)) == (1, 5)          # least egress
    with pytest.raises(rs.ReshardError) as e:
        rs.choose_source([], [], (0, 0))
    assert e.value.name == "NoSource"


def test_plan_cost_examples(rs):
    """single Move of a full F32[4,6] -> 96 bytes each side."""
    cat = rs.Catalog.from_entries([("x", 0, (4, 6), -1, 0)])
    p = rs.generate_plan(cat.build_strategy([(0, 0)], 1, 1, 1), cat.build_strategy([(1, 0)], 1, 1, 1))
    assert p.cost() == {(0, 0): (0, 96), (1, 0): (96, 0)}
    assert p.text() == "MOVE t=x r=[0:4,0:6] 0:0 -> 1:0 bytes=96\n"


def test_catalog_mismatch(rs):
    c1 = rs.Catalog.from_entries([("x", 0, (4,), -1, 0)])
    c2 = rs.Catalog.from_entries([("x", 0, (8,), -1, 0)])
    with pytest.raises(rs.ReshardError) as e:
        rs.generate_plan(c1.build_strategy(DEV(1), 1, 1, 1), c2.build_strategy(DEV(1), 1, 1, 1))
    assert e.value.name == "CatalogMismatch"


def test_fanout_sources_read_once_config3(rs):
    """on a planning-only 8-GPU context for BASELINE configs[2] (GPT-3
    6.7B (4,2,1)->(2,2,2)), the bytes the executing GPUs read (rs_executor_read_bytes summed
    over GPUs) equal the source boxes read ONCE: the union of the Moves' (source device,
    tensor, box) — every DP-replicated fragment feeds both replicas from one read (K3 fan-out
    tiles locally, K2 copy_fan_v16_kernel when a replica is on a peer), and every resident
    relayout fragment is also the source of a Move to the other replica.  Writes are every
    Move and relayout byte once (proj/src/tensor/tensor.cpp:61-78: one slice per source box)."""
    import re

    import bench

    cat, a, b, plan, src_gpu, dst_gpu = bench.build_plan(rs, "gpt3-6.7b-tp4pp2-to-tp2pp2dp2", 8)
    ex = rs.Executor(rs.Context(8, [], []), plan, src_gpu, dst_gpu)
    st = plan.stats()
    boxes = {}
    for ln in plan.text().splitlines():
        if ln.startswith("MOVE"):
            m = re.match(r"MOVE t=(\S+) r=(\S+) (\S+) -> (\S+) bytes=(\d+)", ln)
            boxes[(m.group(3), m.group(1), m.group(2))] = int(m.group(5))
    reads = sum(ex.read_bytes(g) for g in range(8))
    writes = sum(sum(ex.bytes_to(g)) for g in range(8))
    assert reads == sum(boxes.values()) == 93_220_651_008
    assert writes == st["moved_bytes"] + st["relayout_bytes"]  # ~2x: both DP replicas from one read
