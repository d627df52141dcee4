"""SPEC acceptance #6: for the redeployment scenario the central node's
ingress + egress strictly exceeds the maximum per-node traffic of the distributed mode
(qualitative form of the paper's 1.9-2.1x Central/Tenplex claim)."""

DEV = lambda n, w=0: [(w, i) for i in range(n)]  # noqa: E731


def test_redeploy_central_exceeds_distributed(rs):
    cat = rs.Catalog.gpt(64, 4, 16, 128, rs.MIXED_ADAM)
    a = cat.build_strategy(DEV(8), 4, 2, 1)
    b = cat.build_strategy(DEV(8, w=1), 4, 2, 1)
    plan = rs.generate_plan(a, b)
    dist = plan.cost()
    for central in [(0, 0), (1, 3), (2, 0)]:  # a source, a destination, an outside node
        cen = plan.cost_central(central)
        c_io = sum(cen[central])
        assert c_io > max(i + e for i, e in dist.values())
        # conservation: every byte leaves and arrives once per leg
        assert sum(v[0] for v in cen.values()) == sum(v[1] for v in cen.values())


def test_central_same_bytes_per_destination(rs):
    cat = rs.Catalog.gpt(64, 4, 16, 128, rs.FP32_ADAM)
    a = cat.build_strategy(DEV(2), 2, 1, 1)
    b = cat.build_strategy(DEV(4), 2, 1, 2)
    plan = rs.generate_plan(a, b)
    dist, cen = plan.cost(), plan.cost_central((0, 0))
    for d in [(0, 2), (0, 3)]:
        assert cen[d][0] == dist[d][0]  # destinations receive the same bytes either way
    assert sum(cen[(0, 0)]) > max(sum(v) for v in dist.values())
