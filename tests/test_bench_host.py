"""Host-side logic of bench.py (no GPU): catalog windows for waves, the config both arms print,
the whole-workload CPU reference arm (the reference's own compiled slice/merge when
oracle/_ref is built), and the committed K5 traffic figure the dataset line reports."""
import bench
import pytest


def test_windows_cover_the_catalog_in_order(rs):
    cat = rs.Catalog.gpt(4096, 32, 2048, 50304, rs.MIXED_ADAM)
    n = len(cat)
    for waves in range(1, 9):
        wins = bench.windows_of(cat, waves)
        assert wins[0][0] == 0 and wins[-1][1] == n and len(wins) <= waves
        assert all(a < b for a, b in wins) and all(wins[i][1] == wins[i + 1][0] for i in range(len(wins) - 1))
    # equal bytes: no window of the 3-way split holds more than ~half the catalog
    ent = cat.entries()
    per = [bench.WIDTH_OF[e[1]] * __import__("math").prod(e[2]) for e in ent]
    for a, b in bench.windows_of(cat, 3):
        assert sum(per[a:b]) < 0.5 * sum(per)


@pytest.mark.parametrize("name", sorted(bench.WORKLOADS) + sorted(bench.DATASET))
def test_both_arms_print_the_same_config(name):
    """same_config: the reference arm and ours build the dict with the
    same function; it names the workload, the GPU count and the L2 policy."""
    for n in (1, 2, 4, 8):
        c = bench.workload_config(name, n)
        assert c == bench.workload_config(name, n)
        assert c["workload"] == name and c["n_gpus"] == n and "larger than L2" in c["l2"]


def test_cpu_reference_whole_workload_gpt2():
    """The CPU arm times EVERY tensor (no sampling, no scaling by bytes): the bytes it copies per
    step are the plan's moved + relayout bytes, for each threading variant."""
    r = bench.cpu_reference_run("gpt2-small-tp2-to-pp2", 1, 0, variants=("queue", "per_device"))
    plan = r["plan"]
    for v in r["variants"].values():
        assert v["copied_bytes"] == plan["moved_bytes"] + plan["relayout_bytes"]
        assert v["ms"] > 0
    assert r["variants"]["per_device"]["threads"] == 2  # one thread per destination device
    assert "full workload" in r["sample"] and r["host"]["nproc"] >= 1


def test_k5_traffic_from_the_committed_capture():
    assert bench.k5_dram_bytes_per_sample(fused=False) == pytest.approx(173.6, abs=0.5)
    assert bench.k5_dram_bytes_per_sample() == pytest.approx(174.9, abs=0.5)


def test_pcie_overlap_bound():
    """Equal directions: the bidirectional rate alone; a larger side finishes at its one-way rate."""
    link = {"h2d_gbs": 50.0, "d2h_gbs": 40.0, "bidir_gbs_each": 25.0}
    assert bench.pcie_overlap_bound_ms(10**9, 10**9, link) == pytest.approx(40.0)
    assert bench.pcie_overlap_bound_ms(10**9, 3 * 10**9, link) == pytest.approx(40.0 + 50.0)
    assert bench.pcie_overlap_bound_ms(3 * 10**9, 10**9, link) == pytest.approx(40.0 + 40.0)
    assert bench.pcie_overlap_bound_ms(0, 2 * 10**9, link) == pytest.approx(50.0)


def test_windowed_e2e_splits_for_host_ram(rs, monkeypatch):
    """The 6.7B state (94 GB of sources, 188 GB of destinations at N = 1) does not fit the host:
    windowed_e2e picks the fewest catalog windows whose pinned buffers fit the given share of
    host RAM and whose arenas fit the device arenas (planning only here: no GPU calls before
    the split is chosen)."""
    name = "gpt3-6.7b-tp4pp2-to-tp2pp2dp2"
    cat, a, b, plan, src_gpu, dst_gpu = bench.build_plan(rs, name, 1)
    pctx = rs.Context(1, [], [])
    full = rs.Executor(pctx, plan, src_gpu, dst_gpu, 256 << 10).arena_bytes(0)
    monkeypatch.setattr(bench, "host_available_bytes", lambda: 200 * 10**9)

    class Stop(Exception):
        pass

    def no_pinned(n):
        raise Stop(n)

    monkeypatch.setattr(rs, "host_alloc", no_pinned)
    with pytest.raises(Stop) as e:
        bench.windowed_e2e(rs, None, cat, plan, src_gpu, dst_gpu, 256 << 10, full[0], full[1], 0, 0)
    assert e.value.args[0] <= 0.45 * 200 * 10**9 and e.value.args[0] >= full[0] / 8
