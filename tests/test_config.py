"""Parallelization-configuration JSON: examples, round trip through
build_strategy, and planning from parsed documents (identical plans)."""
import json

import pytest

DEV = lambda n: [(0, i) for i in range(n)]  # noqa: E731


def test_two_ranks_half_each(rs):
    """two ranks each declaring half of one [6]-tensor -> sigma {[3]}, 2 partitions."""
    from paper_2312_05181_b200.config import parse_parallel_config

    doc = json.dumps([{"t": {"base": "t", "shape": [6], "range": [[0, 3]], "dtype": "f32"}},
                      {"t": {"base": "t", "shape": [6], "range": [[3, 6]], "dtype": "f32"}}])
    p = parse_parallel_config(doc)
    assert p.hosted_subtensors((0, 0)) == [(0, [(0, 3)])]
    assert p.hosted_subtensors((0, 1)) == [(0, [(3, 6)])]
    assert p.validate() == []
    ref = rs.Catalog.from_entries([("t", 0, (6,), 0, 0)]).build_strategy(DEV(2), 2, 1, 1)
    assert rs.generate_plan(p, ref).text() == ""  # same layout as build_strategy(T=2,P=1,D=1)


def test_errors(rs):
    from paper_2312_05181_b200.config import parse_parallel_config

    def err(doc):
        with pytest.raises(rs.ReshardError) as e:
            parse_parallel_config(doc if isinstance(doc, str) else json.dumps(doc))
        return e.value.name

    leaf = lambda r, shape=(6,), dt="f32": {"base": "t", "shape": list(shape), "range": r, "dtype": dt}  # noqa: E731
    assert err([{"t": leaf([[0, 4]])}, {"t": leaf([[2, 6]])}]) == "CoverageGap"           # SPEC.md:161 overlap
    assert err([{"t": leaf([[0, 2]])}, {"t": leaf([[3, 6]])}]) == "CoverageGap"           # gap
    assert err([{"t": leaf([[0, 3]])}, {"t": leaf([[3, 6]], shape=(7,))}]) == "InconsistentBaseShape"
    assert err([{"t": leaf(None, dt="f64")}]) == "MalformedConfig"
    assert err("[{\"t\": }]") == "MalformedConfig"
    assert err({"t": leaf(None)}) == "MalformedConfig"                                    # not a list
    assert err([{"t": leaf([[0, 9]])}]) == "MalformedConfig"                              # range out of bounds
    # a non-grid rectangulation of a [4,4] tensor is rejected
    two = lambda r: {"base": "m", "shape": [4, 4], "range": r, "dtype": "u8"}  # noqa: E731
    assert err([{"m": two([[0, 2], [0, 4]])}, {"m": two([[2, 4], [0, 2]])}, {"m": two([[2, 4], [2, 4]])}]) == "CoverageGap"


@pytest.mark.parametrize("cfg", [(2, 1, 1), (1, 2, 1), (2, 2, 2), (4, 2, 1), (1, 1, 4)])
def test_round_trip_gpt(rs, cfg):
    from paper_2312_05181_b200.config import parse_parallel_config, serialize_parallel_config

    T, P, D = cfg
    cat = rs.Catalog.gpt(64, 4, 16, 128, rs.MIXED_ADAM)
    orig = cat.build_strategy(DEV(T * P * D), T, P, D)
    doc = serialize_parallel_config(orig)
    ranks = json.loads(doc)
    assert len(ranks) == T * P * D
    assert "layers" in ranks[0] or "embedding" in ranks[0]
    back = parse_parallel_config(doc)
    for d in DEV(T * P * D):
        assert back.hosted_subtensors(d) == orig.hosted_subtensors(d)
    assert serialize_parallel_config(back) == doc
    # plans from / to the parsed layout are the plans of the built layout
    other = cat.build_strategy(DEV(8), 2, 2, 2)
    assert rs.generate_plan(back, other).text() == rs.generate_plan(orig, other).text()
    assert rs.generate_plan(other, back).text() == rs.generate_plan(other, orig).text()
    assert rs.generate_plan(back, orig).text() == ""


def test_custom_devices(rs):
    from paper_2312_05181_b200.config import parse_parallel_config, serialize_parallel_config

    cat = rs.Catalog.gpt(64, 2, 16, 128, rs.FP32_PARAM)
    orig = cat.build_strategy([(1, 0), (1, 1)], 2, 1, 1)
    back = parse_parallel_config(serialize_parallel_config(orig), devices=[(1, 0), (1, 1)])
    assert back.hosted_subtensors((1, 1)) == orig.hosted_subtensors((1, 1))
    with pytest.raises(rs.ReshardError) as e:
        parse_parallel_config(serialize_parallel_config(orig), devices=[(1, 0)])
    assert e.value.name == "DeviceCountMismatch"
