"""Dataset index repartitioning: host functions vs the oracle (CPU), the
SPEC examples and acceptance #8, and the K5 GPU kernel vs the oracle's gather (gpu)."""
import os
import random

import numpy as np
import pytest


def corpus(n, n_files, rng, varlen=True):
    per = (n + n_files - 1) // n_files
    k = np.arange(n, dtype=np.uint64)
    files = k // np.uint64(per)
    lens = (np.array([rng.randint(1, 9000) for _ in range(n)], np.uint64) if varlen
            else np.full(n, 8206, np.uint64))
    offs = np.zeros(n, np.uint64)
    for f in range(n_files):
        sel = files == f
        offs[sel] = np.concatenate([[0], np.cumsum(lens[sel])[:-1]]).astype(np.uint64) if sel.any() else offs[sel]
    return np.stack([files, offs, lens], axis=1).copy()


def classes(n_files, dp, d):
    f = np.arange(n_files)
    m = f % (dp + 1)
    return np.where(m == d, 0, np.where(m == dp, 2, 1)).astype(np.uint8)


def test_shuffle_matches_oracle(rs, orc):
    for n, seed, ep in [(1, 0, 0), (8, 7, 1), (1000, 0x5EED, 0), (54321, 3, 9)]:
        p = rs.shuffle_epoch(n, seed, ep)
        assert np.array_equal(p, orc.shuffle_epoch(n, seed, ep))
        assert np.array_equal(np.sort(p), np.arange(n, dtype=np.uint64))
    assert not np.array_equal(rs.shuffle_epoch(64, 1, 0), rs.shuffle_epoch(64, 1, 1))
    assert rs.shuffle_epoch(1, 5, 5).tolist() == [0]


def test_repartition_examples_and_errors(rs, orc):
    # N=16, B=4, at_step=2, dp 2->4: batch 2 gives ranks {8},{9},{10},{11}
    assert [rs.repartition_position(16, 4, 2, 4, d, 0) for d in range(4)] == [8, 9, 10, 11]
    assert [rs.repartition_count(16, 4, 2, 4, d) for d in range(4)] == [2, 2, 2, 2]
    assert rs.repartition_count(16, 4, 0, 1, 0) == 16
    assert [rs.repartition_count(16, 4, 4, 2, d) for d in range(2)] == [0, 0]
    for args in [(17, 4, 1, 2), (103, 8, 3, 4), (5, 4, 0, 2), (10, 4, 2, 4)]:
        n, B, at, dp = args
        for d in range(dp):
            c = rs.repartition_count(n, B, at, dp, d)
            assert [rs.repartition_position(n, B, at, dp, d, k) for k in range(c)] == \
                list(orc.repartition_positions(n, B, at, dp, d))

    def err(fn):
        with pytest.raises(rs.ReshardError) as e:
            fn()
        return e.value.name

    assert err(lambda: rs.repartition_count(16, 6, 0, 4, 0)) == "IndivisibleBatch"
    assert err(lambda: rs.repartition_count(16, 4, 5, 2, 0)) == "StepBeyondEpoch"
    assert err(lambda: rs.repartition_count(16, 4, 0, 2, 2)) == "IndexOutOfRange"
    assert err(lambda: rs.repartition_position(16, 4, 2, 4, 0, 2)) == "IndexOutOfRange"


def test_locate_sample_priority(rs, orc):
    rng = random.Random(1)
    n, nf = 500, 7
    samples = corpus(n, nf, rng)
    perm = rs.shuffle_epoch(n, 9, 0)
    for dp in (1, 2, 4):
        for d in range(dp):
            fc = classes(nf, dp, d)
            for k in range(0, rs.repartition_count(n, 20, 3, dp, d), 7):
                got = rs.locate_sample(n, 20, 3, dp, d, k, perm, samples, fc)
                assert got == orc.locate_sample(n, 20, 3, dp, d, k, perm, samples, fc)
                assert got[3] == fc[got[0]]


def test_acceptance8_exactly_once_under_dp_changes(rs):
    """SPEC acceptance #8: N <= 10,000, B <= 64, dp changed mid-epoch at 3 random steps:
    the concatenated global read order equals the permutation, each position once."""
    rng = random.Random(8)
    for trial in range(20):
        B = rng.choice([8, 16, 32, 64])
        n = rng.randint(B, 10_000)
        perm = rs.shuffle_epoch(n, 1234 + trial, trial)
        batches = (n + B - 1) // B
        steps = sorted(rng.sample(range(1, batches), min(3, batches - 1)))
        dps = [d for d in (1, 2, 4, 8) if B % d == 0]
        dp = rng.choice(dps)
        order = []
        edges = [0] + steps + [batches]
        for seg in range(len(edges) - 1):
            at, end = edges[seg], edges[seg + 1]
            parts = [[rs.repartition_position(n, B, at, dp, d, k) for k in range(rs.repartition_count(n, B, at, dp, d))]
                     for d in range(dp)]
            b = B // dp
            # replay global order: batch by batch, rank slices in rank order
            ptr = [0] * dp
            for i in range(at, end):
                for d in range(dp):
                    take = [p for p in parts[d][ptr[d]:ptr[d] + b] if p < (i + 1) * B]
                    ptr[d] += len(take)
                    order += [int(perm[p]) for p in take]
            dp = rng.choice(dps)  # B constant, b recomputed
        assert order == [int(x) for x in perm]


@pytest.mark.gpu
@pytest.mark.parametrize("mode,eb", [("split2", 24), ("split2", 32), ("split2_6", 32), ("split2_8", 24),
                                     ("lookback", 24), ("lookback4", 24)])
def test_k5_kernel_matches_oracle(rs, orc, ctx, mode, eb, monkeypatch):
    """K5 against the oracle's restated repartition + locate on ragged
    partitions, trailing partial batches and at_step 0, for every variant and both device
    layouts of the index (packed 24-byte reference records, padded 32-byte)."""
    monkeypatch.setenv("RESHARD_K5", mode)
    rng = random.Random(42)
    for n, nf, B, at, dp in [(50_000, 13, 64, 100, 4), (12_345, 5, 40, 7, 8), (4096, 3, 16, 256, 2),
                             (4096, 3, 16, 0, 1), (300_017, 29, 128, 500, 4)]:
        samples = corpus(n, nf, rng)
        perm = rs.shuffle_epoch(n, n, 1)
        d_perm, d_samp = ctx.malloc(0, 8 * n), ctx.malloc(0, 24 * n)
        ctx.htod(0, d_perm, perm.ctypes.data, 8 * n)
        ctx.htod(0, d_samp, samples.ctypes.data, 24 * n)
        d_idx = d_samp
        if eb == 32:
            d_idx = ctx.malloc(0, 32 * n)
            rs.dataset_index_pad(ctx, 0, d_samp, d_idx, n)
        for d in range(dp):
            fc = classes(nf, dp, d)
            d_fc = ctx.malloc(0, nf)
            ctx.htod(0, d_fc, fc.ctypes.data, nf)
            cnt = rs.repartition_count(n, B, at, dp, d)
            part = rs.Partition(ctx, 0, cnt)
            t = rs.repartition(ctx, 0, d_perm, d_idx, d_fc, n, B, at, dp, d, part, entry_bytes=eb)
            got = part.fetch()
            want = orc.dataset_gather(n, B, at, dp, d, perm, samples, fc, n_threads=3)
            assert np.array_equal(got["pos"], want["pos"])
            assert np.array_equal(got["ent"], want["ent"])
            assert np.array_equal(got["boff"], want["boff"])
            assert got["qcount"] == want["qcount"]
            assert np.array_equal(got["qidx"], want["qidx"])
            assert (t["launches"] > 0) == (cnt > 0)
            part.free()
            ctx.free(0, d_fc)
        ctx.free(0, d_perm)
        ctx.free(0, d_samp)
        if eb == 32:
            ctx.free(0, d_idx)


@pytest.mark.gpu
@pytest.mark.parametrize("eb,fuse", [(24, True), (32, True), (32, False)])
def test_k5_batch_matches_oracle(rs, orc, ctx, eb, fuse, monkeypatch):
    """rs_repartition_batch (a GPU hosting several new DP ranks; fused: one launch per pass for
    every rank, else gather passes back to back and each rank's scan + finalize on a second
    stream) against the oracle:
    every rank of two DP events over one index, incl. empty ranks (at_step past the last full
    batch) and ragged partitions, each with its own locator classes."""
    monkeypatch.setenv("RESHARD_K5_FUSE", "1" if fuse else "0")
    rng = random.Random(77)
    for n, nf, B, events in [(50_000, 13, 64, [(100, 4), (300, 8)]), (12_345, 5, 40, [(7, 8), (0, 2), (308, 4)]),
                             (300_017, 29, 128, [(500, 4), (1000, 8), (2000, 2)]),
                             (40_000, 11, 64, [(0, 8), (200, 8), (400, 4)])]:  # 20 ranks: two launch chunks
        samples = corpus(n, nf, rng)
        perm = rs.shuffle_epoch(n, n, 3)
        d_perm, d_samp = ctx.malloc(0, 8 * n), ctx.malloc(0, 24 * n)
        ctx.htod(0, d_perm, perm.ctypes.data, 8 * n)
        ctx.htod(0, d_samp, samples.ctypes.data, 24 * n)
        d_idx = d_samp
        if eb == 32:
            d_idx = ctx.malloc(0, 32 * n)
            rs.dataset_index_pad(ctx, 0, d_samp, d_idx, n)
        jobs, fcs, held = [], [], []
        for at, dp in events:
            for d in range(dp):
                fc = classes(nf, dp, d)
                d_fc = ctx.malloc(0, nf)
                ctx.htod(0, d_fc, fc.ctypes.data, nf)
                part = rs.Partition(ctx, 0, rs.repartition_count(n, B, at, dp, d))
                jobs.append((at, dp, d, d_fc, part))
                fcs.append(fc)
        t = rs.repartition_batch(ctx, 0, d_perm, d_idx, n, B, jobs, entry_bytes=eb)
        nonempty = sum(1 for j in jobs if j[4].count)
        # fused (default): one launch per pass per chunk of <= 16 ranks; RESHARD_K5_FUSE=0: three per rank
        assert t["launches"] == (3 * ((nonempty + 15) // 16) if fuse else 3 * nonempty)
        assert len(t["per_job"]) == len(jobs) and t["ms"] > 0
        for (at, dp, d, d_fc, part), fc in zip(jobs, fcs):
            got = part.fetch()
            want = orc.dataset_gather(n, B, at, dp, d, perm, samples, fc, n_threads=3)
            assert np.array_equal(got["pos"], want["pos"])
            assert np.array_equal(got["ent"], want["ent"])
            assert np.array_equal(got["boff"], want["boff"])
            assert got["qcount"] == want["qcount"]
            assert np.array_equal(got["qidx"], want["qidx"])
            part.free()
            ctx.free(0, d_fc)
        ctx.free(0, d_perm)
        ctx.free(0, d_samp)
        if eb == 32:
            ctx.free(0, d_idx)


@pytest.mark.gpu
def test_index_pad_layout_and_errors(rs, ctx, monkeypatch):
    """rs_dataset_index_pad writes {file, offset, length, 0} per record; bad entry_bytes and
    the look-back variant on a padded index fail with InvalidArgument."""
    rng = random.Random(5)
    n = 100_003
    samples = corpus(n, 7, rng)
    d_samp, d_pad = ctx.malloc(0, 24 * n), ctx.malloc(0, 32 * n)
    ctx.htod(0, d_samp, samples.ctypes.data, 24 * n)
    t = rs.dataset_index_pad(ctx, 0, d_samp, d_pad, n)
    assert t["launches"] == 1 and t["bytes"] == 32 * n
    got = np.empty((n, 4), np.uint64)
    ctx.dtoh(0, got.ctypes.data, d_pad, 32 * n)
    assert np.array_equal(got[:, :3], samples) and not got[:, 3].any()
    perm = rs.shuffle_epoch(n, 1, 0)
    d_perm, d_fc = ctx.malloc(0, 8 * n), ctx.malloc(0, 7)
    ctx.htod(0, d_perm, perm.ctypes.data, 8 * n)
    fc = classes(7, 2, 0)
    ctx.htod(0, d_fc, fc.ctypes.data, 7)
    part = rs.Partition(ctx, 0, rs.repartition_count(n, 64, 3, 2, 0))
    with pytest.raises(rs.ReshardError, match="InvalidArgument"):
        rs.repartition(ctx, 0, d_perm, d_pad, d_fc, n, 64, 3, 2, 0, part, entry_bytes=16)
    monkeypatch.setenv("RESHARD_K5", "lookback")
    with pytest.raises(rs.ReshardError, match="InvalidArgument"):
        rs.repartition(ctx, 0, d_perm, d_pad, d_fc, n, 64, 3, 2, 0, part, entry_bytes=32)
    part.free()
    for p in (d_samp, d_pad, d_perm, d_fc):
        ctx.free(0, p)


@pytest.mark.gpu
@pytest.mark.parametrize("eb", [24, 32])
def test_host_buffer_path_matches_oracle(rs, orc, ctx, eb):
    """rs_dataset_index_upload + rs_repartition_to_host: pinned host index in, pinned host
    outputs back, equal to the oracle for every rank of a DP change."""
    import ctypes

    rng = random.Random(11)
    n, nf, B, at, dp = 77_777, 11, 96, 40, 4
    samples = corpus(n, nf, rng)
    perm = rs.shuffle_epoch(n, 3, 2)
    h_perm, h_samp = rs.host_alloc(8 * n), rs.host_alloc(24 * n)
    ctypes.memmove(h_perm, perm.ctypes.data, 8 * n)
    ctypes.memmove(h_samp, samples.ctypes.data, 24 * n)
    d_perm, d_samp = ctx.malloc(0, 8 * n), ctx.malloc(0, 24 * n)
    d_pad = ctx.malloc(0, 32 * n) if eb == 32 else 0
    up = rs.dataset_index_upload(ctx, 0, h_perm, h_samp, n, d_perm, d_samp, d_pad)
    assert up["bytes"] == 32 * n and up["launches"] == (1 if eb == 32 else 0)
    for d in range(dp):
        fc = classes(nf, dp, d)
        d_fc = ctx.malloc(0, nf)
        ctx.htod(0, d_fc, fc.ctypes.data, nf)
        cnt = rs.repartition_count(n, B, at, dp, d)
        part, host = rs.Partition(ctx, 0, cnt), rs.HostPartition(cnt)
        r = rs.repartition_to_host(ctx, 0, d_perm, d_pad or d_samp, d_fc, n, B, at, dp, d, part, host, entry_bytes=eb)
        got = host.arrays()
        want = orc.dataset_gather(n, B, at, dp, d, perm, samples, fc, n_threads=2)
        assert np.array_equal(got["pos"], want["pos"]) and np.array_equal(got["ent"], want["ent"])
        assert np.array_equal(got["boff"], want["boff"]) and got["qcount"] == want["qcount"]
        assert np.array_equal(got["qidx"], want["qidx"])
        assert r["d2h_bytes"] == 24 + 40 * cnt + 4 * sum(want["qcount"])
        host.free()
        part.free()
        ctx.free(0, d_fc)
    for p in (d_perm, d_samp) + ((d_pad,) if d_pad else ()):
        ctx.free(0, p)
    rs.host_free(h_perm)
    rs.host_free(h_samp)


def _k8_rounds(n, seed, epoch, window):
    """Round-level restatement of K8's schedule (csrc/cuda/dataset.cu, shuffle_win_*): windowed
    active sets, reservations packed into the high word of the permutation entry (atomicMax of
    i), winners storing their swapped values with the high word cleared, losers carried.  A
    kernel round is this function's round: winners touch disjoint locations and losers do not
    write, so the order of threads inside a launch cannot change the outcome (checked below:
    the losers stay losers when the winners' stores are visible)."""
    gamma, mask = np.uint64(0x9E3779B97F4A7C15), np.uint64(0xFFFFFFFF)

    def draws(i):  # H[i] = splitmix64 draw number n-1-i mod (i+1), i as uint64 array
        with np.errstate(over="ignore"):
            z = np.uint64(seed ^ epoch) + (np.uint64(n) - i) * gamma
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
        return z % (i + np.uint64(1))

    a = np.arange(n, dtype=np.uint64)
    carried, lo, rounds = np.empty(0, np.uint64), n - 1, 0
    while carried.size or lo:
        take = min(max(window - carried.size, 0), lo)
        i = np.concatenate([carried, np.arange(lo, lo - take, -1, dtype=np.uint64)])
        lo -= take
        h = draws(i)
        hi = a >> np.uint64(32)
        np.maximum.at(hi, i.astype(np.int64), i)
        np.maximum.at(hi, h.astype(np.int64), i)
        a = (a & mask) | (hi << np.uint64(32))
        def wins(arr):
            return ((arr[i.astype(np.int64)] >> np.uint64(32)) == i) & ((arr[h.astype(np.int64)] >> np.uint64(32)) == i)

        win = wins(a)
        wi, wh = i[win].astype(np.int64), h[win].astype(np.int64)
        vi, vh = a[wi] & mask, a[wh] & mask
        a[wi], a[wh] = vh, vi  # h == i: both writes store the same value
        # inside a launch a check may see winners' stores (values with the key cleared) or not:
        # the winner set must be the same either way (a rule accepting a cleared key would not be)
        assert np.array_equal(wins(a)[~win], np.zeros((~win).sum(), bool))
        carried = i[~win]
        rounds += 1
    return a, rounds


def test_k8_schedule_restatement_matches_host_shuffle(rs):
    """The packed-reservation, windowed schedule K8 runs is the sequential Fisher-Yates: a
    finished iteration leaves no key behind, so no stale reservation can block or reorder."""
    for n, seed, ep, w in [(2, 3, 1, 1), (3, 7, 0, 1), (1000, 0x5EED, 0, 7), (1000, 0x5EED, 0, 1000),
                           (20_000, 9, 4, 125), (65_537, 2, 2, 65_536), (200_000, 1, 3, 1250)]:
        got, rounds = _k8_rounds(n, seed, ep, w)
        assert np.array_equal(got, rs.shuffle_epoch(n, seed, ep)), (n, w)
        assert rounds >= (n - 1 + w - 1) // w


@pytest.mark.gpu
def test_k8_gpu_shuffle_bit_identical(rs, orc, ctx):
    # 65_536 / 65_537: the window (64 Ki minimum) covers all or all but one iteration; 3M runs
    # many 6-round graph batches with the window 64 Ki
    for n, seed, ep in [(1, 3, 0), (2, 3, 1), (3, 7, 0), (1000, 0x5EED, 0), (65_536, 1, 1), (65_537, 2, 2),
                        (123_457, 9, 4), (3_000_000, 0x5EED, 2)]:
        p = ctx.malloc(0, 8 * n)
        t = rs.shuffle_epoch_device(ctx, 0, n, seed, ep, p)
        got = np.empty(n, np.uint64)
        ctx.dtoh(0, got.ctypes.data, p, 8 * n)
        assert np.array_equal(got, rs.shuffle_epoch(n, seed, ep)), n
        if n <= 200_000:  # and directly against the oracle's restated Fisher-Yates
            assert np.array_equal(got, orc.shuffle_epoch(n, seed, ep)), n
        assert n < 3 or t["rounds"] >= 1
        ctx.free(0, p)


@pytest.mark.gpu
def test_config5_full_size_matches_oracle(rs, orc, ctx):
    """BASELINE config 5 at full size (N = 10^8, B = 1280, DP 2 -> 4 -> 8): the K8 GPU epoch
    permutation equals the host Fisher-Yates, and every rank's K5 output (positions, entries,
    byte offsets, locator queues) equals the oracle's gather on the same inputs (17 tile-scan
    blocks per rank; the 2 -> 4 event reads the packed index, 4 -> 8 the padded one)."""
    n, B, files, per_file, sb = 100_000_000, 1280, 1000, 100_000, 8206
    k = np.arange(n, dtype=np.uint64)
    samples = np.empty((n, 3), np.uint64)
    samples[:, 0] = k // np.uint64(per_file)
    samples[:, 1] = (k % np.uint64(per_file)) * np.uint64(sb)
    samples[:, 2] = sb
    del k
    perm = rs.shuffle_epoch(n, 0x5EED, 0)
    assert np.array_equal(perm, orc.shuffle_epoch(n, 0x5EED, 0))  # the host loop is the oracle's
    d_perm, d_samp = ctx.malloc(0, 8 * n), ctx.malloc(0, 24 * n)
    ctx.htod(0, d_samp, samples.ctypes.data, 24 * n)
    rs.shuffle_epoch_device(ctx, 0, n, 0x5EED, 0, d_perm)
    dev_perm = np.empty(n, np.uint64)
    ctx.dtoh(0, dev_perm.ctypes.data, d_perm, 8 * n)
    assert np.array_equal(dev_perm, perm)
    del dev_perm
    d_pad = ctx.malloc(0, 32 * n)
    rs.dataset_index_pad(ctx, 0, d_samp, d_pad, n)
    for (at, dp), eb in [((25_000, 4), 24), ((50_000, 8), 32)]:  # packed then padded index
        for d in range(dp):
            m = np.arange(files) % (dp + 1)
            fc = np.where(m == d, 0, np.where(m == dp, 2, 1)).astype(np.uint8)
            d_fc = ctx.malloc(0, files)
            ctx.htod(0, d_fc, fc.ctypes.data, files)
            part = rs.Partition(ctx, 0, rs.repartition_count(n, B, at, dp, d))
            rs.repartition(ctx, 0, d_perm, d_pad if eb == 32 else d_samp, d_fc, n, B, at, dp, d, part, entry_bytes=eb)
            got = part.fetch()
            want = orc.dataset_gather(n, B, at, dp, d, perm, samples, fc, n_threads=os.cpu_count() or 1)
            for key in ("pos", "ent", "boff", "qidx"):
                assert np.array_equal(got[key], want[key]), (at, dp, d, key)
            assert got["qcount"] == want["qcount"]
            del got, want
            part.free()
            ctx.free(0, d_fc)
    ctx.free(0, d_perm)
    ctx.free(0, d_samp)
    ctx.free(0, d_pad)
