#!/usr/bin/env python
"""Reshard benchmark: PTC state transformation on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl ours|reference]

A step is one apply_plan of the workload's reconfiguration over state already resident
in HBM (synthetic random-init payload of the named model shapes), started from a barrier.
`value` is the reshard time in ms: from one common start to the last GPU's completion (CUDA
events; one process driving N GPUs) or, under torchrun (one process per GPU), each rank's
event time from a per-step barrier, max over ranks.  `e2e` is the same metric through the
C-ABI with host buffers (H2D of the source arenas from pinned memory, the reshard kernels,
D2H of the destination arenas).  Inputs (>= 18 GB) exceed the 126 MB L2, so no flush is
needed between steps.  Logical device d lives on GPU d % N; cross-GPU fragments are pushed
over NVLink by the source GPU's kernels (peer stores into the destination's arena).

    python bench.py --gpus N            one process, N GPUs (peer access), needs N devices —
                                        or RESHARD_SAME_GPU=1: the N-GPU world emulated on cuda:0
    torchrun ... bench.py --gpus N      one process per GPU, dst arenas exchanged by CUDA IPC
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "reshard time (ms) + effective GB/s vs HBM/NVLink roofline for TP/PP/DP A->B"

# name: (catalog args (h, L, S, V, kind), from (T, P, D, devices), to (T, P, D, devices), failed)
WORKLOADS = {
    # BASELINE configs[1]: GPT-3 1.3B bf16+fp32 Adam scale-out (TP2,PP1,DP1)->(TP2,PP1,DP2), 2->4
    "gpt3-1.3b-dp-scaleout": ((2048, 24, 2048, 50304, 1), (2, 1, 1, [0, 1]), (2, 1, 2, [0, 1, 2, 3]), []),
    # configs[0]: GPT-2 small fp32+Adam (TP2,PP1,DP1)->(TP1,PP2,DP1), 2 ranks
    "gpt2-small-tp2-to-pp2": ((768, 12, 1024, 50304, 0), (2, 1, 1, [0, 1]), (1, 2, 1, [0, 1]), []),
    # configs[2]: GPT-3 6.7B (TP4,PP2,DP1)->(TP2,PP2,DP2), 8 GPUs (needs >= 2 GPUs of HBM)
    "gpt3-6.7b-tp4pp2-to-tp2pp2dp2": ((4096, 32, 2048, 50304, 1), (4, 2, 1, list(range(8))),
                                       (2, 2, 2, list(range(8))), []),
    # configs[3]: GPT-3 6.7B failure recovery (TP2,PP2,DP2)->(TP2,PP2,DP1), failed {1,3,4,6}
    "gpt3-6.7b-recovery": ((4096, 32, 2048, 50304, 1), (2, 2, 2, list(range(8))), (2, 2, 1, [0, 2, 5, 7]),
                           [1, 3, 4, 6]),
}
DEFAULT_WORKLOAD = "gpt3-1.3b-dp-scaleout"
WIDTH_OF = {0: 4, 1: 2, 2: 8, 3: 1, 4: 2}  # dtype code -> bytes (F32, F16, I64, U8, BF16)
# configs[4]: dataset index repartition of a 100M-sample corpus under DP 2 -> 4 -> 8
DATASET = {"dataset-100m-dp2to4to8": dict(n=100_000_000, B=1280, seed=0x5EED, epoch=0, files=1000,
                                          per_file=100_000, sample_bytes=8206, events=[(25_000, 4), (50_000, 8)])}
DATASET_BYTES_PER_SAMPLE = 8 + 24 + 8 + 24 + 8 + 4  # read perm+entry, write pos+entry+boff+queue index
# K5's dominant kernel, the gather pass: read perm + entry, write pos + entry + parked length + class byte
DATASET_GATHER_BYTES_PER_SAMPLE = 8 + 24 + 8 + 24 + 8 + 1


def dataset_inputs(spec):
    import numpy as np

    n = spec["n"]
    k = np.arange(n, dtype=np.uint64)
    samples = np.empty((n, 3), np.uint64)
    samples[:, 0] = k // np.uint64(spec["per_file"])
    samples[:, 1] = (k % np.uint64(spec["per_file"])) * np.uint64(spec["sample_bytes"])
    samples[:, 2] = spec["sample_bytes"]
    return samples


def dataset_classes(files, dp, d):
    """Locator class of every file for rank d: round-robin holders, one in dp+1 remote-only."""
    import numpy as np

    m = np.arange(files) % (dp + 1)
    return np.where(m == d, 0, np.where(m == dp, 2, 1)).astype(np.uint8)


def _reduce(dist, local, vals, op):
    """All-reduce a list of floats over the ranks (max or sum); identity for one process."""
    if dist is None:
        return vals
    import torch

    t = torch.tensor(vals, dtype=torch.float64, device=f"cuda:{local}" if DIST_BACKEND == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return [float(x) for x in t.tolist()]


def run_dataset(args, rs, dist=None):
    """configs[4]: every new DP rank's repartition of both events; rank d of an event runs on
    GPU d % N (each GPU independent, no data-path collective: scaling "weak" in ranks per
    GPU, the time is the max over GPUs of their ranks' device time)."""
    import numpy as np

    rank, world, local = dist_env()
    spec = DATASET[args.workload]
    n = spec["n"]
    t_host = time.perf_counter()
    perm = rs.shuffle_epoch(n, spec["seed"], spec["epoch"])  # host reference of the epoch order
    host_shuffle_ms = (time.perf_counter() - t_host) * 1e3
    samples = dataset_inputs(spec)
    ctx = rs.Context(world, [rank], [local])
    d_perm, d_samp = ctx.malloc(rank, 8 * n), ctx.malloc(rank, 24 * n)
    ctx.htod(rank, d_samp, samples.ctypes.data, 24 * n)
    # device layout of the static index: padded 32-byte records (one per sector), written once
    # per index load by rs_dataset_index_pad; RESHARD_INDEX=packed keeps the 24-byte records
    eb = 24 if os.environ.get("RESHARD_INDEX", "padded") == "packed" else 32
    d_idx, pad_ms = d_samp, None
    if eb == 32:
        d_idx = ctx.malloc(rank, 32 * n)
        pad_ms = rs.dataset_index_pad(ctx, rank, d_samp, d_idx, n)["ms"]
    # K8: the epoch permutation on the GPU (bit-identical to the host shuffle, checked here)
    shuf = [rs.shuffle_epoch_device(ctx, rank, n, spec["seed"], spec["epoch"], d_perm) for _ in range(2)][-1]
    dev_perm = np.empty(n, np.uint64)
    ctx.dtoh(rank, dev_perm.ctypes.data, d_perm, 8 * n)
    shuffle_identical = bool(np.array_equal(dev_perm, perm))
    del dev_perm
    jobs = []  # (at_step, dp, d, class ptr, partition)
    for at, dp in spec["events"]:
        for d in range(dp):
            if d % world != rank:
                continue
            fc = dataset_classes(spec["files"], dp, d)
            p_fc = ctx.malloc(rank, spec["files"])
            ctx.htod(rank, p_fc, fc.ctypes.data, spec["files"])
            jobs.append((at, dp, d, p_fc, rs.Partition(ctx, rank, rs.repartition_count(n, spec["B"], at, dp, d))))

    # this GPU's ranks in one batch: one launch per pass for all of them (default), or with
    # RESHARD_K5_FUSE=0 the gather passes back to back and each rank's scan + finalize on a
    # second stream; RESHARD_K5_BATCH=0: one rs_repartition call per rank
    batched = os.environ.get("RESHARD_K5_BATCH", "1") != "0"
    fused = batched and os.environ.get("RESHARD_K5_FUSE", "1") != "0"
    k5_schedule = ("rs_repartition_batch, fused: every rank of this GPU in one launch per pass (gather, tile scan, "
                   "finalize)" if fused else
                   "rs_repartition_batch: the ranks' gather passes back to back, each rank's scan + finalize on a "
                   "low-priority second stream" if batched else "rs_repartition per rank, one after another")

    def step():
        if batched:
            t = rs.repartition_batch(ctx, rank, d_perm, d_idx, n, spec["B"], jobs, entry_bytes=eb)
            return t["ms"], t["gather_ms"], sum(j[4].count for j in jobs), t["launches"]
        ms, gms, samples_done, launches = 0.0, 0.0, 0, 0
        for at, dp, d, p_fc, part in jobs:
            t = rs.repartition(ctx, rank, d_perm, d_idx, p_fc, n, spec["B"], at, dp, d, part, entry_bytes=eb)
            ms += t["ms"]
            gms += t["gather_ms"]
            samples_done += part.count
            launches += t["launches"]
        return ms, gms, samples_done, launches

    for _ in range(args.warmup):
        step()
    ctx.sync(rank)
    if dist is not None:
        dist.barrier()
    step_ms, gather_ms = [], []
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            ms, gms, done, launches = step()
            step_ms.append(ms)
            gather_ms.append(gms)
    ctx.sync(rank)
    if dist is not None:
        dist.barrier()
    # parity spot check of the last step against the host restatement: every rank of this GPU,
    # ~1,000 sampled positions and entries each
    pos_ok, ent_ok = True, True
    for at, dp, d, _, part in jobs:
        got = part.fetch()
        stride = max(1, part.count // 1000)
        pos_ok = pos_ok and all(int(got["pos"][k]) == rs.repartition_position(n, spec["B"], at, dp, d, k)
                                for k in range(0, part.count, stride))
        ent_ok = ent_ok and bool(np.array_equal(got["ent"][::stride], samples[perm[got["pos"][::stride]]]))
        del got
    # the floor of the same step: K5's gathers plus its output stores, no scan (off the clock)
    floor_ms = sum(rs.repartition_gather_probe(ctx, rank, d_perm, d_idx, n, spec["B"], at, dp, d, entry_bytes=eb)["ms"]
                   for at, dp, d, _, _ in jobs)
    e2e = None
    if not args.no_e2e:
        try:
            e2e = dataset_e2e(args, rs, ctx, rank, spec, perm, samples, d_perm, d_samp, d_idx if eb == 32 else 0, eb,
                              jobs)
        except Exception as exc:  # e.g. not enough pinned host memory on this box
            e2e = {"value": None, "unit": "ms", "error": str(exc)[:200], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    # step time: max over GPUs of each GPU's device time; samples / launches summed.  The
    # dominant kernel's achieved GB/s is per GPU: all GPUs' gather bytes over all GPUs'
    # gather-pass time (the average launch of the dominant kernel).
    split2 = os.environ.get("RESHARD_K5", "split2").startswith("split2")
    per_sample = DATASET_GATHER_BYTES_PER_SAMPLE if split2 else DATASET_BYTES_PER_SAMPLE
    # ranks on their own GPUs run concurrently: the step is the slowest GPU's time; ranks sharing
    # one GPU (RESHARD_SAME_GPU emulation) are time-sliced on it: the step is the sum of their times
    shared = dist is not None and bool(os.environ.get("RESHARD_SAME_GPU"))
    ms, floor_ms = _reduce(dist, local, [statistics.mean(step_ms), floor_ms], "sum" if shared else "max")
    done_r = done
    done, launches, g_sum, b_sum = _reduce(dist, local, [done, launches, statistics.mean(gather_ms), done_r * per_sample],
                                           "sum")
    done, launches = int(done), int(launches)
    if e2e is not None and dist is not None:  # every rank takes part in the same collectives
        ok = e2e["value"] is not None
        failed, v = _reduce(dist, local, [0.0 if ok else 1.0, e2e["value"] if ok else 0.0], "max")
        h2d, d2h = _reduce(dist, local, [e2e["h2d_bytes_per_step"], e2e["d2h_bytes_per_step"]], "sum")
        if failed:
            e2e = {"value": None, "unit": "ms", "error": e2e.get("error", "failed on another rank"),
                   "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
        else:
            e2e["value"] = round(v, 3)
            e2e["h2d_bytes_per_step"], e2e["d2h_bytes_per_step"] = int(h2d), int(d2h)
            e2e["note"] = "per GPU: upload of the whole index, its ranks' K5 + D2H; max over GPUs"
            e2e.pop("roofline", None)
    if rank != 0:
        return
    peak, peak_kind = measured_peaks()
    alg = done * DATASET_BYTES_PER_SAMPLE
    gms = g_sum / world  # mean over GPUs of the gather-pass time per step
    galg = done * per_sample
    achieved = b_sum / (g_sum * 1e-3) / 1e9  # the dominant kernel (gather pass) over its own event time
    n_gather = max(1, launches // 3)  # gather launches per step: one per rank, or one per batch (fused)
    dram_ps = k5_dram_bytes_per_sample(fused)
    traffic = round(dram_ps * done / n_gather) if dram_ps and split2 else None
    line = {
        "metric": METRIC, "value": round(ms, 4), "unit": "ms", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (100M-sample index, 1000 files)",
        "config": workload_config(args.workload, args.gpus),
        "index_layout": "padded 32-byte records" if eb == 32 else "packed 24-byte records",
        "k5_schedule": k5_schedule,
        "index_pad_ms_once": None if pad_ms is None else round(pad_ms, 3),
        "samples_per_step": done, "gsamples_per_s": round(done / (ms * 1e-3) / 1e9, 3),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic, "peak_kind": peak_kind, "peak_how": peak_how(),
                     "dram_bytes_per_sample": dram_ps,
                     "dram_frac": round(dram_ps * (b_sum / per_sample) / (g_sum * 1e-3) / 1e9 / peak, 4) if dram_ps else None,
                     "traffic_note": "ncu dram read+write of the gather pass per sample (profiles/r2_35/k5_fused_ncu.json; "
                                     "per-rank launches: r2_03/k5_sectors.json) x samples per launch: a random 32-byte "
                                     "record costs a whole 128-byte DRAM line",
                     "kernel": ("repart_gather2_multi_kernel" if fused else "repart_gather2_kernel") if split2
                     else "repartition_kernel",
                     "algorithmic_bytes_per_launch": galg // max(n_gather, 1),
                     "kernel_ms_per_step": round(gms, 4),
                     "step_achieved_gbs": round(alg / (ms * 1e-3) / 1e9, 1),
                     "gather_write_floor_ms": round(floor_ms, 4),
                     "kernel_frac_of_floor": round(floor_ms / gms, 4) if world == 1 else None,
                     "step_frac_of_floor": round(floor_ms / ms, 4),
                     "floor_note": "gather_write_probe_kernel, one launch per rank: the same perm + entry gathers "
                                   "and the 44 output bytes per sample, coalesced, no scan (its per-rank launch tails "
                                   "are part of it, the fused batch has none); random 24-B gathers cost whole DRAM "
                                   "lines, so the streaming-HBM frac is not reachable"},
        "gpu_launches": launches * args.steps, "clocks": clocks.summary(), "spot_check": {"pos": pos_ok, "ent": ent_ok},
        "emulation": AUTO_EMULATED or (f"{world} ranks share cuda:0 (step = the sum of their device times)"
                                       if world > 1 and os.environ.get("RESHARD_SAME_GPU") else None),
        "e2e": e2e,
        "shuffle_epoch_gpu": {"ms": round(shuf["ms"], 3), "rounds": shuf["rounds"], "launches": shuf["launches"],
                              "bit_identical_to_host": shuffle_identical,
                              "host_shuffle_ms_1thread": round(host_shuffle_ms, 1)},
    }
    if not args.no_cpu_baseline and world == 1:
        from oracle.oracle import Oracle

        o = Oracle()
        threads = os.cpu_count() or 1
        secs = 0.0
        for at, dp in spec["events"]:
            for d in range(dp):
                r = o.dataset_gather(n, spec["B"], at, dp, d, perm, samples, dataset_classes(spec["files"], dp, d),
                                     n_threads=threads)
                secs += r["seconds"]
                del r
        line["cpu_baseline"] = {"value": round(secs * 1e3, 3), "unit": "ms", "cores": threads, "kind": "port",
                                "sample": "full workload (all ranks of both DP events), restated gather with "
                                          f"{threads} threads"}
    print(json.dumps(line), flush=True)


def dataset_e2e(args, rs, ctx, rank, spec, perm, samples, d_perm, d_samp, d_pad, eb, jobs):
    """The dataset step through the C ABI with host buffers: every step uploads the epoch
    permutation and the packed index from pinned memory (and pads it on the device), runs
    every rank's K5, and reads every rank's outputs back into pinned buffers.  Wall clock
    around the whole step (each call returns after its stream work)."""
    import ctypes

    import numpy as np

    n = spec["n"]
    h_perm, h_samp = rs.host_alloc(8 * n), rs.host_alloc(24 * n)
    ctypes.memmove(h_perm, perm.ctypes.data, 8 * n)
    ctypes.memmove(h_samp, samples.ctypes.data, 24 * n)
    hosts = [rs.HostPartition(part.count) for *_, part in jobs]
    try:
        step_ms, d2h = [], 0
        for i in range(1 + args.e2e_steps):  # the first pass warms up the pinned pages
            t0 = time.perf_counter()
            up = rs.dataset_index_upload(ctx, rank, h_perm, h_samp, n, d_perm, d_samp, d_pad)
            d2h = 0
            for (at, dp, d, p_fc, part), host in zip(jobs, hosts):
                r = rs.repartition_to_host(ctx, rank, d_perm, d_pad or d_samp, p_fc, n, spec["B"], at, dp, d, part,
                                           host, entry_bytes=eb)
                d2h += r["d2h_bytes"]
            if i:
                step_ms.append((time.perf_counter() - t0) * 1e3)
        # the host copies agree with the device outputs
        at, dp, d, _, part = jobs[-1]
        got, want = hosts[-1].arrays(), part.fetch()
        same = all(np.array_equal(got[k], want[k]) for k in ("pos", "ent", "boff", "qidx")) and \
            got["qcount"] == want["qcount"]
        line = {"value": round(statistics.mean(step_ms), 3), "unit": "ms", "h2d_bytes_per_step": up["bytes"],
                "d2h_bytes_per_step": d2h, "steps": args.e2e_steps, "host_matches_device": bool(same),
                "path": "rs_dataset_index_upload + rs_repartition_to_host per rank, pinned host buffers"}
        try:
            if dist_env()[1] > 1:
                raise RuntimeError("PCIe roofline measured in one-GPU runs only")
            link = pcie_probe()
            bound = up["bytes"] / (link["h2d_gbs"] * 1e9) * 1e3 + d2h / (link["d2h_gbs"] * 1e9) * 1e3
            line["roofline"] = {"bound": "pcie", **link, "bound_ms": round(bound, 2),
                                "frac": round(bound / line["value"], 4),
                                "note": "H2D then D2H at the measured one-way rates (the gathers need the whole "
                                        "index before any output exists)"}
        except Exception as exc:  # noqa: BLE001
            line["roofline"] = {"error": str(exc)[:200]}
        return line
    finally:
        for h in hosts:
            h.free()
        rs.host_free(h_perm)
        rs.host_free(h_samp)


DIST_BACKEND = os.environ.get("RESHARD_DIST_BACKEND", "nccl")


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    if os.environ.get("RESHARD_SAME_GPU"):  # every rank on cuda:0 (IPC correctness on one GPU)
        local = 0
    return rank, world, local


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def peak_how() -> str:
    """How the driver measured the HBM peak (MEASURED_PEAKS.json `how`): a torch copy_ of a
    few GiB, read + write bytes — a copy kernel streaming tens of GB can exceed it (frac > 1)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            how = str(json.load(f).get("how", ""))
        # the HBM clause only (the file also describes the bf16 matmul peak)
        return next((c.strip() for c in how.split(";") if "copy" in c), how)[:200]
    except Exception:
        return "fallback: /opt/skills/guides/B200_PROFILING.md"


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {
        0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting", 0x1: "gpu_idle",
    }

    def __init__(self, cuda_index: int, period_s: float = 0.005):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        self.period = period_s
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[cuda_index]) if vis else cuda_index
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _loop(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._loop, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def pcie_probe(nbytes: int = 2 << 30, reps: int = 6) -> dict:
    """Pinned host <-> device copy rates on this box (off the clock): the link that bounds the
    host-buffer e2e path.  H2D alone, D2H alone, and both directions at once on two streams."""
    import torch

    h_in = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h_out = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d_a = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(ops):
        best = float("inf")
        for _ in range(reps):
            torch.cuda.synchronize()
            ev = []
            for stream, fn in ops:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                with torch.cuda.stream(stream):
                    fn()
                e1.record(stream)
                ev.append((e0, e1))
            torch.cuda.synchronize()
            best = min(best, max(a.elapsed_time(b) for a, b in ev))
        return best

    h2d = lambda: d_a.copy_(h_in, non_blocking=True)  # noqa: E731
    d2h = lambda: h_out.copy_(d_b, non_blocking=True)  # noqa: E731
    t_h2d = timed([(s1, h2d)])
    t_d2h = timed([(s2, d2h)])
    t_both = timed([(s1, h2d), (s2, d2h)])
    del h_in, h_out, d_a, d_b
    torch.cuda.empty_cache()
    gb = nbytes / 1e9
    return {"h2d_gbs": round(gb / (t_h2d * 1e-3), 1), "d2h_gbs": round(gb / (t_d2h * 1e-3), 1),
            "bidir_gbs_each": round(gb / (t_both * 1e-3), 1), "probe_bytes": nbytes}


def pcie_overlap_bound_ms(h2d: int, d2h: int, link: dict) -> float:
    """Lower bound of a pipeline that moves h2d bytes up and d2h bytes down at once: both
    directions at the measured bidirectional rate until the smaller side is done, then the rest
    of the larger side at its one-way rate."""
    lo, hi = min(h2d, d2h), max(h2d, d2h)
    alone = link["h2d_gbs"] if h2d >= d2h else link["d2h_gbs"]
    return (lo / (link["bidir_gbs_each"] * 1e9) + (hi - lo) / (alone * 1e9)) * 1e3


def copy_kernel_name(tiles_per_launch: int = 0) -> str:
    """The dominant copy kernel: the library default is bulk_strided, which a launch of at least
    RESHARD_DYN_MIN_TILES (2e5) tiles runs as bulk_dyn (dynamic claims)."""
    k = os.environ.get("RESHARD_COPY_KERNEL", "bulk_strided") or "bulk_strided"  # the library default
    dyn_min = int(os.environ.get("RESHARD_DYN_MIN_TILES", "200000") or 0)
    if k == "bulk_strided" and dyn_min > 0 and tiles_per_launch >= dyn_min and \
            os.environ.get("RESHARD_BULK_HINT", "0") in ("", "0"):
        k = "bulk_dyn"
    return {"bulk": "copy_bulk_kernel", "bulk_strided": "copy_bulk_strided_kernel", "ldg": "copy_v16_kernel",
            "ldg8": "copy_v16_kernel", "bulk_warp": "copy_bulk_warp_kernel", "bulk_dyn": "copy_bulk_dyn_kernel"}.get(k, k)


def k5_dram_bytes_per_sample(fused: bool = True):
    """DRAM read + write bytes per sample of K5's gather pass (committed ncu captures: the fused
    multi-rank launch, profiles/r2_35; one rank's launch, profiles/r2_03)."""
    try:
        if fused:
            with open(os.path.join(ROOT, "profiles", "r2_35", "k5_fused_ncu.json")) as f:
                v = json.load(f)
        else:
            with open(os.path.join(ROOT, "profiles", "r2_03", "k5_sectors.json")) as f:
                v = json.load(f)["variants"]["ldg"]
        return round(v["dram_read_bytes_per_sample"] + v["dram_write_bytes_per_sample"], 1)
    except Exception:
        return None


def ncu_traffic(workload: str, kernel: str):
    """dram read+write bytes per launch of `kernel` from the committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "ncu_copy_tiles.json")
    try:
        with open(p) as f:
            d = json.load(f)
        e = d.get(workload, {}).get(kernel)
        return None if e is None else float(e["dram_bytes_per_launch"])
    except Exception:
        return None


def build_plan(rs, name, n_gpus):
    (h, L, S, V, kind), (T1, P1, D1, devs1), (T2, P2, D2, devs2), failed = WORKLOADS[name]
    cat = rs.Catalog.gpt(h, L, S, V, kind)
    a = cat.build_strategy([(0, d) for d in devs1], T1, P1, D1)
    b = cat.build_strategy([(0, d) for d in devs2], T2, P2, D2)
    t0 = time.perf_counter()
    plan = rs.recover(a, [(0, d) for d in failed], b) if failed else rs.generate_plan(a, b)
    build_plan.plan_ms = (time.perf_counter() - t0) * 1e3  # Alg. 1 on the host (reported apart)
    src_gpu = [d % n_gpus for d in devs1]
    dst_gpu = [d % n_gpus for d in devs2]
    return cat, a, b, plan, src_gpu, dst_gpu


def workload_config(name: str, n_gpus: int, mode: str = "distributed") -> dict:
    """The `config` both arms print for a workload (identical dicts: same_config)."""
    if name in DATASET:
        spec = DATASET[name]
        return {"workload": name, "events": spec["events"], "B": spec["B"], "n": spec["n"], "n_gpus": n_gpus,
                "placement": "new DP rank d on GPU d % n_gpus", "l2": "inputs larger than L2 (no flush)"}
    _, (T1, P1, D1, devs1), (T2, P2, D2, devs2), failed = WORKLOADS[name]
    return {"workload": name, "transition": f"(TP{T1},PP{P1},DP{D1})->(TP{T2},PP{P2},DP{D2})",
            "failed_devices": failed, "logical_devices": max(len(devs1), len(devs2)), "n_gpus": n_gpus,
            "placement": "logical device d on GPU d % n_gpus", "mode": mode, "l2": "inputs larger than L2 (no flush)"}


def host_info() -> dict:
    """CPU model, core count and RAM of this host (SURVEY §8d / BASELINE.md §3)."""
    model, ram = None, None
    try:
        with open("/proc/cpuinfo") as f:
            model = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), None)
        with open("/proc/meminfo") as f:
            kb = next(int(ln.split()[1]) for ln in f if ln.startswith("MemTotal"))
        ram = round(kb / 2**20, 1)
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "ram_gib": ram}


def host_available_bytes() -> int:
    try:
        with open("/proc/meminfo") as f:
            return next(int(ln.split()[1]) for ln in f if ln.startswith("MemAvailable")) * 1024
    except Exception:
        return 0


# ---------------------------------------------------------------------------------------
def cpu_reference_run(name: str, steps: int, warmup: int, variants=("queue",), dst_budget_gb: float = 48.0) -> dict:
    """The reference's CPU path on this host over the WHOLE workload: the SPEC-restated
    planner/executor over the reference's own compiled slice()/merge() (oracle/_ref/libptc_ref.so;
    the restated oracle, kind "port", when that build is absent).  The source state is filled once
    (off the clock); the catalog is applied in windows whose destination state fits next to it in
    host RAM (GPT-3 6.7B: SURVEY §8d's "stream per base tensor"), and a step's time is the sum of
    the windows' apply times (steady_clock inside orc_apply: barrier 1 to barrier 2).
    Variants: "queue" — every host core drains a shared (destination, tensor, cell) queue (the
    headline); "per_device" — one thread per destination device, capped at nproc;
    "1thread" — one thread (one step)."""
    from oracle.oracle import Oracle, lib_path

    ref = os.path.exists(lib_path(True))
    o = Oracle(reference=ref)
    (h, L, S, V, kind), (T1, P1, D1, devs1), (T2, P2, D2, devs2), failed = WORKLOADS[name]
    cat = o.catalog_gpt(h, L, S, V, kind)
    a = cat.build_strategy([(0, d) for d in devs1], T1, P1, D1)
    b = cat.build_strategy([(0, d) for d in devs2], T2, P2, D2)
    plan = a.plan(b, failed=[(0, d) for d in failed])
    st = plan.stats()
    ent = cat.entries()
    per_t = []
    for _, dt, shape, _, _ in ent:
        n = WIDTH_OF[dt]
        for e in shape:
            n *= e
        per_t.append(n)
    ratio = st["dst_bytes"] / max(sum(per_t), 1)  # destination bytes per base byte
    windows, t0, acc = [], 0, 0
    for t, nb in enumerate(per_t):
        if acc and (acc + nb) * ratio > dst_budget_gb * 1e9:
            windows.append((t0, t))
            t0, acc = t, 0
        acc += nb
    windows.append((t0, len(per_t)))
    tf = time.perf_counter()
    src = a.fill(skip=[(0, d) for d in failed])  # a recovery's failed devices hold nothing
    fill_s = time.perf_counter() - tf
    threads = os.cpu_count() or 1
    n_dst_dev = len(devs2)

    def one_step(n_threads, per_device):
        secs, moved = 0.0, 0
        for w0, w1 in windows:
            out, rep = plan.apply(src, n_threads=n_threads, t0=w0, t1=w1, per_device=per_device)
            del out
            secs += rep["seconds"]
            moved += rep["moved"] + rep["local"]
        return secs * 1e3, moved

    res = {}
    for v in variants:
        nt, pd, k, wu = {"queue": (threads, False, steps, warmup),
                         "per_device": (min(threads, n_dst_dev), True, max(1, min(steps, 3)), 0),
                         "1thread": (1, False, 1, 0)}[v]
        ms = []
        for i in range(wu + k):
            t, moved = one_step(nt, pd)
            if i >= wu:
                ms.append(t)
        res[v] = {"ms": round(statistics.mean(ms), 3), "threads": nt, "steps": k, "ms_samples": [round(x, 3) for x in ms],
                  "copied_bytes": moved}
    del src
    head = res[variants[0]]
    return {
        "value": head["ms"], "ms_samples": head["ms_samples"], "unit": "ms", "cores": head["threads"],
        "kind": "reference" if ref else "port",
        "sample": (f"full workload: all {len(per_t)} tensors, {head['copied_bytes'] / 1e9:.2f} GB copied per step "
                   f"in {len(windows)} catalog window(s) over one filled source state; "
                   f"{head['threads']} threads draining destination cells"),
        "variants": res, "host": host_info(), "fill_s_once": round(fill_s, 2),
        "plan": {k: st[k] for k in ("n_move", "n_merge", "moved_bytes", "relayout_bytes")},
    }


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    if args.workload in DATASET:
        import paper_2312_05181_b200 as rs
        from oracle.oracle import Oracle

        spec = DATASET[args.workload]
        perm = rs.shuffle_epoch(spec["n"], spec["seed"], spec["epoch"])
        samples = dataset_inputs(spec)
        o, threads, ms = Oracle(), os.cpu_count() or 1, []
        for i in range(args.warmup + args.steps):
            secs = 0.0
            for at, dp in spec["events"]:
                for d in range(dp):
                    secs += o.dataset_gather(spec["n"], spec["B"], at, dp, d, perm, samples,
                                             dataset_classes(spec["files"], dp, d), n_threads=threads)["seconds"]
            if i >= args.warmup:
                ms.append(secs * 1e3)
        leg = {"value": statistics.mean(ms), "cores": threads, "kind": "port",
               "sample": f"full workload, restated gather (oracle.cpp orc_dataset_gather), {threads} threads",
               "host": host_info()}
    else:
        leg = cpu_reference_run(args.workload, args.steps, args.warmup, variants=("queue",))
    line = {
        "impl": "reference", "metric": METRIC, "value": round(leg["value"], 3), "unit": "ms",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(leg["value"], 3),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "dtype": "u64" if args.workload in DATASET else "u8",
        "data": "synthetic (100M-sample index, 1000 files)" if args.workload in DATASET
        else "synthetic (splitmix64 payload of the model shapes)",
        "config": workload_config(args.workload, args.gpus, args.mode),
        "cpu_baseline": {"value": round(leg["value"], 3), "unit": "ms", "cores": leg["cores"], "kind": leg["kind"],
                         "sample": leg["sample"], "host": leg["host"]},
        "e2e": {"value": round(leg["value"], 3), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------
def gpu_map(rs, n_gpus: int):
    """World GPU -> CUDA device for a single-process N-GPU world: one device per world GPU when
    the box has N, else (RESHARD_SAME_GPU=1) every world GPU on cuda:0 — the correctness
    emulation of an N-GPU world on one device (its peer stores are local stores)."""
    n = rs.device_count()
    if n >= n_gpus:
        return list(range(n_gpus)), False
    if os.environ.get("RESHARD_SAME_GPU"):
        return [0] * n_gpus, True
    raise SystemExit(f"--gpus {n_gpus}: {n} CUDA device(s) visible (RESHARD_SAME_GPU=1 emulates the world on cuda:0)")


def windows_of(cat, waves: int):
    """Catalog windows of ~equal bytes (waves: executed one after another over reused arenas)."""
    ent = cat.entries()
    per_t = []
    for e in ent:
        n = WIDTH_OF[e[1]]
        for x in e[2]:
            n *= x
        per_t.append(n)
    total_b, bounds, acc = sum(per_t), [0], 0
    for t, nb in enumerate(per_t):
        acc += nb
        if len(bounds) < waves and acc >= total_b * len(bounds) / waves:
            bounds.append(t + 1)
    bounds.append(len(ent))
    return [(bounds[i], bounds[i + 1]) for i in range(len(bounds) - 1) if bounds[i + 1] > bounds[i]]


def p2p_probe(rs, ctx, cuda_of, nbytes: int = 1 << 30, reps: int = 3) -> dict:
    """Measured NVLink peer bandwidth on this box (off the clock; distinct GPUs only).
    pair_sm: our K1 LDG/STG kernel on GPU 0 storing 1 GiB into GPU 1's memory (rs_broadcast,
    SM stores over NVLink); pair_ce / ring_ce: copy-engine peer copies (torch), GPU 0 -> 1 alone
    and every GPU -> the next one at once.  `peak` = the best per-GPU one-way rate seen."""
    import torch

    n = len(cuda_of)
    out = {"probe_bytes": nbytes}
    src = ctx.malloc(0, nbytes)
    dst = ctx.malloc(1, nbytes)
    old = os.environ.get("RESHARD_COPY_KERNEL")
    os.environ["RESHARD_COPY_KERNEL"] = "ldg"
    try:
        ms = min(rs.broadcast(ctx, 0, src, [dst], nbytes)["ms"] for _ in range(reps))
        out["pair_sm_gbs"] = round(nbytes / (ms * 1e-3) / 1e9, 1)
    finally:
        if old is None:
            os.environ.pop("RESHARD_COPY_KERNEL", None)
        else:
            os.environ["RESHARD_COPY_KERNEL"] = old
        ctx.free(0, src)
        ctx.free(1, dst)
    bufs = [(torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{c}"),
             torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{c}")) for c in cuda_of]

    def timed(pairs):
        best = float("inf")
        for _ in range(reps):
            for c in cuda_of:
                torch.cuda.synchronize(c)
            ev = []
            for s, d in pairs:
                with torch.cuda.device(cuda_of[s]):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    bufs[d][1].copy_(bufs[s][0], non_blocking=True)
                    e1.record()
                ev.append((e0, e1))
            for c in cuda_of:
                torch.cuda.synchronize(c)
            best = min(best, max(a.elapsed_time(b) for a, b in ev))
        return best

    out["pair_ce_gbs"] = round(nbytes / (timed([(0, 1)]) * 1e-3) / 1e9, 1)
    out["ring_ce_gbs_per_gpu"] = round(nbytes / (timed([(g, (g + 1) % n) for g in range(n)]) * 1e-3) / 1e9, 1)
    del bufs
    torch.cuda.empty_cache()
    out["peak"] = max(out["pair_sm_gbs"], out["pair_ce_gbs"], out["ring_ce_gbs_per_gpu"])
    return out


def pinned_total(dist, local, nbytes: int) -> int:
    """Pinned host bytes every rank of the world would allocate (all ranks call this)."""
    import torch

    t = torch.tensor([float(nbytes)], dtype=torch.float64, device=f"cuda:{local}" if DIST_BACKEND == "nccl" else "cpu")
    dist.all_reduce(t)
    return int(t.item())


def windowed_e2e(rs, ctx, cat, plan, src_gpu, dst_gpu, tile, src_b, dst_b, src_ptr, dst_ptr,
                 host_frac: float = 0.45) -> dict:
    """The step end to end from pinned host buffers when the whole state does not fit the host
    (GPT-3 6.7B: 94 GB of sources + 188 GB of destinations vs ~200 GB of host RAM) or the GPU
    (waves): the catalog in the fewest host windows whose pinned src + dst buffers fit
    `host_frac` of the available host RAM and whose arenas fit the device arenas already bound;
    per window the sources are filled on the device and copied to the host buffer (off the
    clock), one warm-up rs_executor_run_host (pins the pages, plans the host chunks), then one
    timed run_host: H2D | copy kernel | D2H of that window.  value = sum over windows."""
    avail = host_available_bytes()
    pctx = rs.Context(1, [], [])
    wins = None
    for k in range(1, 65):
        cand = windows_of(cat, k)
        sizes = [rs.Executor(pctx, plan, src_gpu, dst_gpu, tile, window=w if len(cand) > 1 else None).arena_bytes(0)
                 for w in cand]
        if all(s <= src_b and d <= dst_b for s, d in sizes) and max(s + d for s, d in sizes) <= host_frac * avail:
            wins = cand
            break
    if wins is None:
        raise RuntimeError("no host window split fits the host RAM and the device arenas")
    hs_b, hd_b = max(s for s, _ in sizes), max(d for _, d in sizes)
    hs, hd = rs.host_alloc(max(hs_b, 1)), rs.host_alloc(max(hd_b, 1))
    ms, ms_full, bad, h2d, d2h, per = 0.0, 0.0, 0, 0, 0, []
    try:
        for w, (s, d) in zip(wins, sizes):
            ex = rs.Executor(ctx, plan, src_gpu, dst_gpu, tile, window=w if len(wins) > 1 else None)
            ex.bind(0, src_ptr, dst_ptr)
            ex.prepare()
            ex.fill_sources()
            ctx.dtoh(0, hs, src_ptr, s)
            ex.run_host(0, hs, hd, skip_unread=True)
            t = ex.run_host(0, hs, hd, skip_unread=True)["ms"]
            bad += ex.verify()
            up = ex.host_upload_bytes(0, skip_unread=True)
            t_full = ex.run_host(0, hs, hd)["ms"]  # the same with the whole src arena uploaded
            ms, h2d, d2h, ms_full = ms + t, h2d + up, d2h + d, ms_full + t_full
            per.append({"window": list(w), "ms": round(t, 2), "h2d": up, "d2h": d, "src_arena": s,
                        "ms_full_src_upload": round(t_full, 2)})
            del ex
    finally:
        rs.host_free(hs)
        rs.host_free(hd)
    return {"value": round(ms, 3), "unit": "ms", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": 1,
            "mismatched_bytes": bad, "windows": per, "host_buffers_gb": round((hs_b + hd_b) / 1e9, 1),
            "ms_full_src_upload": round(ms_full, 3),
            "path": f"rs_executor_run_host_flags(RS_HOST_SKIP_UNREAD) per host window ({len(wins)} catalog windows, "
                    "sum of the windows' H2D of the source ranges the tiles read | copy kernel | D2H times; the "
                    "whole state exceeds host RAM; cells kept in place stay in the host buffer)"}


def world_e2e(rs, plan, src_gpu, dst_gpu, n_gpus, cuda_devs, tile, steps) -> dict:
    """The step end to end from pinned host buffers through rs_executor_run_host_world, one
    process driving every GPU (own context, arenas and executor; sources filled with K6 and
    copied to the host buffers first, off the clock)."""
    ctx = rs.Context(n_gpus, list(range(n_gpus)), list(cuda_devs))
    ex = rs.Executor(ctx, plan, src_gpu, dst_gpu, tile)
    ex.allocate_local()
    ex.prepare()
    ex.fill_sources()
    hs, hd, s_tot, d_tot = [], [], 0, 0
    try:
        for g in range(n_gpus):
            s_b, d_b = ex.arena_bytes(g)
            s_tot, d_tot = s_tot + s_b, d_tot + d_b
            hs.append(rs.host_alloc(max(s_b, 1)))
            hd.append(rs.host_alloc(max(d_b, 1)))
            ctx.dtoh(g, hs[g], ex.arenas[g][0], s_b)
        ex.run_host_world(hs, hd)
        ms = [ex.run_host_world(hs, hd) for _ in range(steps)]
        bad = ex.verify()
    finally:
        for p in hs + hd:
            rs.host_free(p)
        del ex
    return {"value": round(statistics.mean(ms), 3), "unit": "ms", "h2d_bytes_per_step": s_tot, "d2h_bytes_per_step": d_tot,
            "steps": steps, "mismatched_bytes": bad,
            "path": "rs_executor_run_host_world from one process driving every GPU: pipelined rounds of H2D | "
                    "pushes | D2H (RESHARD_WORLD_PIPELINE=0: three phases)"}


def run_ours(args):
    import paper_2312_05181_b200 as rs

    rank, world, local = dist_env()
    N = args.gpus
    if world > 1 and world != N:
        raise SystemExit(f"--gpus {N} but WORLD_SIZE={world}")
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist

        if DIST_BACKEND == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:  # gloo plumbing: lets several ranks share one GPU (multi-process correctness runs)
            dist.init_process_group("gloo")
    if args.workload in DATASET:
        return run_dataset(args, rs, dist)
    cat, a, b, plan, src_gpu, dst_gpu = build_plan(rs, args.workload, N)
    # the world GPUs this process drives: its own (one process per GPU, torchrun), or all N
    if world > 1:
        mine, cuda_of, emulated = [rank], [local], bool(os.environ.get("RESHARD_SAME_GPU"))
    else:
        mine = list(range(N))
        cuda_of, emulated = gpu_map(rs, N)
    ctx = rs.Context(N, mine, cuda_of)
    tile = args.tile_kib << 10

    # waves: the fewest catalog windows whose arenas fit each CUDA device (180 GB HBM3e each)
    import torch

    budget = {}
    for c in set(cuda_of):
        free, _ = torch.cuda.mem_get_info(c)
        budget[c] = int(free * 0.92) // (N if (world > 1 and emulated) else 1)
    pctx = rs.Context(N, [], [])  # planning-only view: layouts, no device work
    windows, s_need, d_need = None, None, None
    for waves in ([args.waves] if args.waves else range(1, 9)):
        wins = windows_of(cat, waves)
        pexs = [rs.Executor(pctx, plan, src_gpu, dst_gpu, tile, window=w if len(wins) > 1 else None) for w in wins]
        s_need = {g: max(p.arena_bytes(g)[0] for p in pexs) for g in mine}
        d_need = {g: max(p.arena_bytes(g)[1] for p in pexs) for g in mine}
        per_dev = {}
        for g, c in zip(mine, cuda_of):
            per_dev[c] = per_dev.get(c, 0) + s_need[g] + d_need[g]
        del pexs
        windows = wins
        if all(per_dev[c] <= budget[c] for c in per_dev):
            break
    if args.mode == "central" and (world > 1 or len(windows) > 1):
        raise SystemExit("--mode central: single-process, single-wave workloads only")
    t_lower = time.perf_counter()
    if args.mode == "central":
        exs = [rs.Executor(ctx, plan, src_gpu, dst_gpu, tile, central=0)]
    else:
        exs = [rs.Executor(ctx, plan, src_gpu, dst_gpu, tile, window=w if len(windows) > 1 else None) for w in windows]
    lower_ms = (time.perf_counter() - t_lower) * 1e3  # arena layout + fragments -> pieces (host)
    src_ptr, dst_ptr = {}, {}
    for g in mine:
        s_b = max(e.arena_bytes(g)[0] for e in exs)
        d_b = max(e.arena_bytes(g)[1] for e in exs)
        s_need[g], d_need[g] = s_b, d_b
        src_ptr[g], dst_ptr[g] = ctx.malloc(g, max(s_b, 256)), ctx.malloc(g, max(d_b, 256))
        for ex in exs:
            ex.bind(g, src_ptr[g], dst_ptr[g])
    if dist is not None:
        # destination arenas of every GPU, mapped into this process (CUDA IPC over NVLink)
        handle = ctx.ipc_handle(rank, dst_ptr[rank]) if d_need[rank] else None
        handles = [None] * world
        dist.all_gather_object(handles, handle)
        for g in range(world):
            if g != rank and handles[g] is not None:
                p = ctx.ipc_open(rank, handles[g])
                for ex in exs:
                    ex.bind(g, 0, p)
    t_prep = time.perf_counter()
    for ex in exs:
        ex.prepare()  # bind bases into the pieces, upload them; the GPU expands them into tiles
    prepare_ms = (time.perf_counter() - t_prep) * 1e3
    if len(exs) == 1:
        exs[0].fill_sources()
    stats = plan.stats()

    def barrier():
        for g in mine:
            ctx.sync(g)
        if dist is not None:
            dist.barrier()

    # one process per GPU: a common start and the last rank's end on the device, through
    # interprocess events — rank 0 records start + "go", every other rank's stream waits on "go"
    # before its kernels and records its "done", rank 0's stream waits on every "done" and records
    # the end (SPEC.md:501's two barriers; host barriers only order the enqueues)
    if dist is not None:
        go = rs.Event(ctx, rank, "ipc") if rank == 0 else None
        done = rs.Event(ctx, rank, "ipc")
        handles = [None] * world
        dist.all_gather_object(handles, (go.handle if go else None, done.handle))
        if rank == 0:
            peers_done = [rs.Event(ctx, 0, "ipc", handles[r][1]) for r in range(1, world)]
            t_start, t_end = rs.Event(ctx, 0), rs.Event(ctx, 0)
        else:
            go_peer = rs.Event(ctx, rank, "ipc", handles[0][0])

    def step(verify=False):
        """One reshard: every wave from a barrier (every GPU idle, every rank here), timed from
        one common start to the last GPU's completion (single process: world events; one
        process per GPU: interprocess events into rank 0's timeline; the max over ranks of each
        rank's own kernel time beside it)."""
        ms, gpu_ms, bad, launches = 0.0, 0.0, 0, 0
        for ex in exs:
            if len(exs) > 1:
                ex.fill_sources()  # the window's sources (off the clock)
            barrier()
            if dist is not None:
                if rank == 0:
                    t_start.record()
                    go.record()
                dist.barrier()  # "go" is enqueued before anyone waits on it
                if rank != 0:
                    go_peer.wait()
                ex.run()
                done.record()
                dist.barrier()  # every "done" is enqueued before rank 0 waits on them
                if rank == 0:
                    for e in peers_done:
                        e.wait()
                    t_end.record()
                t = ex.wait()
                ms += t_end.elapsed_since(t_start) if rank == 0 else 0.0
            else:
                ex.run()
                t = ex.wait()
                ms += ex.world_ms()
            gpu_ms += max(x["ms"] for x in t)
            launches += sum(x["launches"] for x in t)
            if verify and len(exs) > 1:
                barrier()  # every peer's pushes of this wave landed before anyone checks it
                bad += ex.verify()
        return ms, gpu_ms, bad, launches

    for _ in range(args.warmup):
        step()
    barrier()
    step_ms, gpu_step_ms, launches_total, bad_w = [], [], 0, 0
    with ClockSampler(cuda_of[0]) as clocks:
        t0 = time.perf_counter()
        for i in range(args.steps):
            ms_i, g_i, b_i, l_i = step(verify=(i == args.steps - 1))
            step_ms.append(ms_i)
            gpu_step_ms.append(g_i)
            launches_total += l_i
            bad_w += b_i
        barrier()
        wall = time.perf_counter() - t0
    if dist is not None:  # per step: rank 0's world time; the slowest rank's own kernel time beside it
        dev = f"cuda:{local}" if DIST_BACKEND == "nccl" else "cpu"
        tt = torch.tensor(step_ms + gpu_step_ms, dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        step_ms = [float(x) for x in tt[:args.steps].tolist()]
        gpu_step_ms = [float(x) for x in tt[args.steps:].tolist()]
        lt = torch.tensor([float(launches_total)], dtype=torch.float64, device=dev)
        dist.all_reduce(lt)
        launches_total = int(lt.item())
    ms = statistics.mean(step_ms)
    bad = exs[0].verify() if len(exs) == 1 else bad_w
    if dist is not None:
        tb = torch.tensor([bad], device=f"cuda:{local}" if DIST_BACKEND == "nccl" else "cpu", dtype=torch.int64)
        dist.all_reduce(tb)
        bad = int(tb.item())

    # the all-to-all: bytes each GPU's tiles write into every GPU, and the bytes they read
    rows = [[0] * N for _ in range(N)]
    rbs = [0] * N
    for g in mine:
        rows[g] = [sum(v) for v in zip(*(ex.bytes_to(g) for ex in exs))]
        rbs[g] = sum(ex.read_bytes(g) for ex in exs)
    if dist is not None:
        dev = f"cuda:{local}" if DIST_BACKEND == "nccl" else "cpu"
        m = torch.tensor(rows, dtype=torch.float64, device=dev)
        rb = torch.tensor(rbs, dtype=torch.float64, device=dev)
        dist.all_reduce(m)
        dist.all_reduce(rb)
        rows = [[int(x) for x in r] for r in m.cpu().tolist()]
        rbs = [int(x) for x in rb.cpu().tolist()]

    # e2e through the C-ABI with host buffers
    ex = exs[0]
    e2e = None
    total_host = sum(s_need.values()) + sum(d_need.values())
    if args.no_e2e:
        e2e = None
    elif (len(exs) > 1 or total_host > 0.6 * host_available_bytes()) and world == 1 and N == 1 \
            and args.mode == "distributed":
        try:
            e2e = windowed_e2e(rs, ctx, cat, plan, src_gpu, dst_gpu, tile, s_need[0], d_need[0], src_ptr[0], dst_ptr[0])
            try:  # the PCIe bound of the same windows, both directions at once within each window
                link = pcie_probe()
                bound_ms = sum(pcie_overlap_bound_ms(w["h2d"], w["d2h"], link) for w in e2e["windows"])
                e2e["roofline"] = {"bound": "pcie", **link, "bound_ms": round(bound_ms, 2),
                                   "frac": round(bound_ms / e2e["value"], 4)}
            except Exception as exc:  # noqa: BLE001
                e2e["roofline"] = {"error": str(exc)[:200]}
        except Exception as exc:  # noqa: BLE001  (e.g. not enough pinned host memory)
            e2e = {"value": None, "unit": "ms", "error": str(exc)[:200]}
    elif len(exs) > 1:
        e2e = {"value": None, "unit": "ms", "note": "waves at N > 1: host-buffer path not run (state exceeds the GPUs' HBM)"}
    elif world == 1:
        if total_host > 0.6 * host_available_bytes():
            e2e = {"value": None, "unit": "ms", "note": f"host buffers of {total_host / 1e9:.1f} GB exceed 60% of host RAM"}
        else:
            hs = {g: rs.host_alloc(max(s_need[g], 1)) for g in mine}
            hd = {g: rs.host_alloc(max(d_need[g], 1)) for g in mine}
            try:
                for g in mine:
                    ctx.dtoh(g, hs[g], src_ptr[g], s_need[g])
                h2d_bytes = sum(s_need.values())
                if N == 1:  # one GPU: the chunk-pipelined host path (H2D | kernels | D2H overlapped)
                    skip = args.mode == "distributed"
                    ex.run_host(0, hs[0], hd[0], skip_unread=skip)
                    e2e_ms = [ex.run_host(0, hs[0], hd[0], skip_unread=skip)["ms"] for _ in range(args.e2e_steps)]
                    h2d_bytes = ex.host_upload_bytes(0, skip_unread=skip)
                    path = ("rs_executor_run_host_flags(RS_HOST_SKIP_UNREAD): chunk-pipelined H2D of the source "
                            "ranges the tiles read | copy kernel | D2H, pinned host buffers") if skip else \
                        "rs_executor_run_host: H2D | kernels | D2H, pinned host buffers"
                else:  # all GPUs from one common start: H2D | world barrier | kernels | barrier | D2H
                    hs_l, hd_l = [hs[g] for g in range(N)], [hd[g] for g in range(N)]
                    ex.run_host_world(hs_l, hd_l)
                    e2e_ms = [ex.run_host_world(hs_l, hd_l) for _ in range(args.e2e_steps)]
                    path = ("rs_executor_run_host_world: pipelined rounds of H2D | pushes | D2H over every GPU "
                            "(RESHARD_WORLD_PIPELINE=0: three phases)")
                bad_e2e = ex.verify()
                d_eff = sum(d_need.values()) - ex.staging_bytes()
                e2e = {"value": round(statistics.mean(e2e_ms), 3), "unit": "ms",
                       "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": d_eff,
                       "steps": args.e2e_steps, "mismatched_bytes": bad_e2e, "path": path}
                if N == 1:
                    try:  # the PCIe bound of this path, measured on the same box
                        link = pcie_probe()
                        if args.mode == "central":  # H2D, both phases, D2H in sequence (no chunk pipeline)
                            bound_ms = (h2d_bytes / (link["h2d_gbs"] * 1e9) + d_eff / (link["d2h_gbs"] * 1e9)) * 1e3
                        else:  # chunk pipeline: both directions at once
                            bound_ms = pcie_overlap_bound_ms(h2d_bytes, d_eff, link)
                        e2e["roofline"] = {"bound": "pcie", **link, "bound_ms": round(bound_ms, 2),
                                           "frac": round(bound_ms / e2e["value"], 4)}
                    except Exception as exc:
                        e2e["roofline"] = {"error": str(exc)[:200]}
            except Exception as exc:  # e.g. not enough pinned host memory
                e2e = {"value": None, "unit": "ms", "h2d_bytes_per_step": sum(s_need.values()),
                       "d2h_bytes_per_step": sum(d_need.values()), "error": str(exc)[:200]}
            finally:
                for g in mine:
                    rs.host_free(hs[g])
                    rs.host_free(hd[g])
    elif pinned_total(dist, local, s_need[rank] + d_need[rank]) > 0.6 * host_available_bytes():
        e2e = {"value": None, "unit": "ms", "note": "pinned host buffers of all ranks exceed 60% of host RAM"}
    else:
        # one process per GPU: H2D of its src arena | barrier | push kernels | barrier | D2H of
        # its dst arena; CUDA events mark to mark on each rank's stream, max over ranks
        hs, hd = rs.host_alloc(max(s_need[rank], 1)), rs.host_alloc(max(d_need[rank], 1))
        ctx.dtoh(rank, hs, src_ptr[rank], s_need[rank])
        e2e_ms = []
        for i in range(1 + args.e2e_steps):
            ex.host_phase(rank, 0, hs)
            dist.barrier()
            ex.host_phase(rank, 1)
            dist.barrier()
            ex.host_phase(rank, 2, hd)
            if i:
                e2e_ms.append(ex.host_elapsed(rank))
        dev = f"cuda:{local}" if DIST_BACKEND == "nccl" else "cpu"
        t = torch.tensor([statistics.mean(e2e_ms)], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        totals = torch.tensor([s_need[rank], d_need[rank]], dtype=torch.int64, device=dev)
        dist.all_reduce(totals)
        rs.host_free(hs)
        rs.host_free(hd)
        e2e = {"value": round(float(t.item()), 3), "unit": "ms", "h2d_bytes_per_step": int(totals[0].item()),
               "d2h_bytes_per_step": int(totals[1].item()), "steps": args.e2e_steps,
               "path": "per rank: H2D | barrier | kernels | barrier | D2H (rs_executor_host_phase), max over ranks"}
        # the same step through the single-process world API (rank 0 drives every GPU of the node,
        # pipelined rounds) while the other ranks wait; the line reports the faster of the two
        dist.barrier()
        world_line = None
        if rank == 0:
            try:
                devs = list(cuda_of) * N if emulated else list(range(N))
                world_line = world_e2e(rs, plan, src_gpu, dst_gpu, N, devs[:N], tile, args.e2e_steps)
            except Exception as exc:  # noqa: BLE001
                world_line = {"error": str(exc)[:200]}
        dist.barrier()
        if rank == 0 and world_line and world_line.get("value") and world_line["mismatched_bytes"] == 0:
            e2e = dict(world_line, per_rank_phases=e2e) if world_line["value"] < e2e["value"] else \
                dict(e2e, world_api=world_line)

    # ExecutionReport verification digests, off the clock (after the e2e runs,
    # which rewrite the same destination bytes): per base tensor the
    # FNV-1a-64 of the tensor reassembled from the destination cells (the LAST DP copy of each, so
    # the copies the reshard wrote are the ones hashed) against the source layout's
    report = None
    if len(exs) == 1 and world == 1 and args.mode == "distributed" and not args.no_digests and \
            sum(s_need.values()) <= 40e9:
        t_d = time.perf_counter()
        d_src, d_dst = exs[0].digests(0), exs[0].digests(1, replica=-1)
        report = {"digest": "fnv1a64 per base tensor", "tensors": len(d_dst), "match": d_src == d_dst and len(d_dst) == len(cat),
                  "seconds": round(time.perf_counter() - t_d, 2)}
    # NVLink peak measured on this box (distinct GPUs only), else the NVLink 5 spec
    p2p = None
    if N > 1 and not emulated and not args.no_p2p_probe:
        if world == 1:
            try:
                p2p = p2p_probe(rs, ctx, cuda_of)
            except Exception as exc:  # noqa: BLE001
                p2p = {"error": str(exc)[:200]}
        else:  # one process per GPU: rank 0 probes every GPU of the node while the others wait
            dist.barrier()
            if rank == 0:
                try:
                    devs = list(range(min(N, torch.cuda.device_count())))
                    p2p = p2p_probe(rs, rs.Context(len(devs), devs, devs), devs)
                except Exception as exc:  # noqa: BLE001
                    p2p = {"error": str(exc)[:200]}
            dist.barrier()
    # the NVLink denominator: the P2P peak measured on this box, else the pool's measured peer copy
    # (B200_PROFILING.md: 770 GB/s per direction; 900 nominal)
    bw_nvl = p2p["peak"] if p2p and "peak" in p2p else 770.0
    bw_nvl_kind = ("measured on this box (p2p_probe)" if p2p and "peak" in p2p
                   else "fallback: B200_PROFILING.md measured peer copy, 770 GB/s per direction (900 nominal)")
    peak, peak_kind = measured_peaks()

    def fabric_of(rows, rbs, n, bw_link):
        """T_roof = max_g max(in_g / BW_nvl, out_g / BW_nvl, hbm_g / BW_hbm)."""
        t_roof, worst, terms = 0.0, None, []
        for g in range(n):
            out_g = sum(rows[g][w] for w in range(n) if w != g)
            in_g = sum(rows[r][g] for r in range(n) if r != g)
            hbm_g = rbs[g] + sum(rows[r][g] for r in range(n))  # reads of its tiles + every write landing in it
            terms.append((out_g, in_g, hbm_g))
            for kind, t in (("nvlink_out", out_g / bw_link), ("nvlink_in", in_g / bw_link), ("hbm", hbm_g / peak)):
                if t / 1e6 > t_roof:
                    t_roof, worst = t / 1e6, {"gpu": g, "term": kind}
        return t_roof, worst, terms

    fabric = None
    if N == 1:  # derived: the same plan over its own GPU count (no such box here)
        n_native = max(len(WORKLOADS[args.workload][1][3]), len(WORKLOADS[args.workload][2][3]))
        if n_native > 1:
            _, _, _, nplan, nsrc, ndst = build_plan(rs, args.workload, n_native)
            pex = rs.Executor(rs.Context(n_native, [], []), nplan, nsrc, ndst, tile)
            rows_n = [pex.bytes_to(g) for g in range(n_native)]
            rbs_n = [pex.read_bytes(g) for g in range(n_native)]
            t_roof, worst, _ = fabric_of(rows_n, rbs_n, n_native, 900.0)
            t_roof_770, _, _ = fabric_of(rows_n, rbs_n, n_native, 770.0)
            fabric = {"derived_for_gpus": n_native, "t_roof_ms": round(t_roof, 3), "bottleneck": worst,
                      "t_roof_ms_at_measured_peer_copy": round(t_roof_770, 3),
                      "note": "not measured: SURVEY 8d's T_roof of this plan on its own GPU count (NVLink 900 GB/s "
                              "per direction nominal; 770 GB/s = the pool's measured peer copy; measured HBM peak), "
                              "for comparison with the 1-GPU emulation above"}
    else:
        t_roof, worst, terms = fabric_of(rows, rbs, N, bw_nvl)
        fabric = {"t_roof_ms": round(t_roof, 3), "frac": round(t_roof / ms, 4) if ms and not emulated else None,
                  "bottleneck": worst, "bw_nvlink_gbs": bw_nvl, "bw_nvlink_kind": bw_nvl_kind, "p2p_probe": p2p,
                  "max_egress_gb": round(max(t[0] for t in terms) / 1e9, 3),
                  "max_ingress_gb": round(max(t[1] for t in terms) / 1e9, 3),
                  "max_hbm_gb": round(max(t[2] for t in terms) / 1e9, 3)}
        if emulated:
            fabric["note"] = ("RESHARD_SAME_GPU: every world GPU on cuda:0 (peer stores are local stores); "
                              "T_roof is the plan's on N real GPUs, not comparable with this time")
    if rank != 0:
        return
    writes = sum(sum(r) for r in rows)
    reads = sum(rbs)
    tiles_all = sum(ex.tiles(g)[0] for ex in exs for g in mine)
    kname = copy_kernel_name(tiles_all // max(1, len(exs) * len(mine)))
    if N == 1 or emulated:
        # every byte on one device: HBM read + write of every copied byte over the step time
        achieved = (reads + writes) / (ms * 1e-3) / 1e9
        traffic = ncu_traffic(args.workload, kname) if args.mode == "distributed" and N == 1 else None
        roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(achieved / peak, 4), "traffic": traffic, "peak_kind": peak_kind, "peak_how": peak_how(),
                    "kernel": kname, "algorithmic_bytes_per_step": reads + writes,
                    "launches_per_step": launches_total // max(args.steps, 1)}
        if emulated:
            roofline["note"] = f"{N} world GPUs emulated on cuda:0: the whole all-to-all is HBM traffic of one device"
    else:
        # the fabric: the busiest GPU's NVLink direction over the world time
        _, _, terms = fabric_of(rows, rbs, N, bw_nvl)
        link = max(max(t[0], t[1]) for t in terms)
        hbm_max = max(t[2] for t in terms)
        achieved = link / (ms * 1e-3) / 1e9
        roofline = {"bound": "nvlink", "achieved": round(achieved, 1), "peak": bw_nvl, "unit": "GB/s",
                    "frac": round(achieved / bw_nvl, 4), "traffic": None, "peak_kind": bw_nvl_kind,
                    "kernel": kname + " + copy_fan_v16_kernel / copy_v16_kernel (peer stores)",
                    "algorithmic_bytes_per_step": {"busiest_link": link, "all_writes": writes, "all_reads": reads},
                    "hbm": {"achieved": round(hbm_max / (ms * 1e-3) / 1e9, 1), "peak": peak,
                            "frac": round(hbm_max / (ms * 1e-3) / 1e9 / peak, 4)},
                    "launches_per_step": launches_total // max(args.steps, 1)}
    line = {
        "metric": METRIC, "value": round(ms, 4), "unit": "ms", "n_gpus": N, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic (splitmix64 payload of the model shapes)",
        "config": workload_config(args.workload, N, args.mode),
        "timing": ("one process: common start event on GPU 0, every GPU waits on it, GPU 0 joins every GPU's end"
                   if world == 1 else "one process per GPU: rank 0's start + interprocess 'go' event every rank waits "
                                      "on, every rank's interprocess 'done' event rank 0 waits on before its end event"),
        "ms_max_gpu_kernel": round(statistics.mean(gpu_step_ms), 4),
        "emulated_on_one_gpu": emulated if N > 1 else None,
        "effective_gbs": round((stats["moved_bytes"] + stats["relayout_bytes"]) / (ms * 1e-3) / 1e9, 1),
        "fabric": fabric,
        "moved_bytes": stats["moved_bytes"], "relayout_bytes": stats["relayout_bytes"],
        "kept_bytes": stats["kept_bytes"], "plan": {k: stats[k] for k in ("n_split", "n_move", "n_merge")},
        "roofline": roofline,
        "e2e": e2e, "gpu_launches": launches_total, "waves": len(exs), "emulation": AUTO_EMULATED,
        "clocks": clocks.summary(), "verify_mismatched_bytes": bad, "execution_report": report, "wall_s": round(wall, 4),
        "ms_min": round(min(step_ms), 4), "ms_median": round(statistics.median(step_ms), 4),
        "tiles": tiles_all,
        "host_ms": {"plan": round(build_plan.plan_ms, 2), "lower": round(lower_ms, 2), "prepare": round(prepare_ms, 2),
                    "reconfiguration_total_ms": round(build_plan.plan_ms + lower_ms + prepare_ms + ms, 2),
                    "note": "off the clock, once per reconfiguration: Alg. 1 planning, arena layout + piece "
                            "lowering, descriptor binding + upload + device expansion"},
    }
    if N == 1 and not args.no_cpu_baseline:
        try:
            variants = ["queue", "per_device"] + (["1thread"] if stats["moved_bytes"] < 40e9 else [])
            leg = cpu_reference_run(args.workload, 2, 1, variants=variants)
            line["cpu_baseline"] = {"value": leg["value"], "unit": "ms", "cores": leg["cores"], "kind": leg["kind"],
                                    "sample": leg["sample"], "variants": leg["variants"], "host": leg["host"]}
        except Exception as exc:
            line["cpu_baseline"] = {"value": None, "error": str(exc)[:200]}
    print(json.dumps(line), flush=True)


def relaunch_under_torchrun(args) -> None:
    """`--gpus N` with no launcher on a per-rank path (the dataset workload): re-exec this
    command under torch.distributed.run, one process per GPU (gloo when RESHARD_SAME_GPU puts
    every rank on cuda:0)."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    if env.get("RESHARD_SAME_GPU"):
        env.setdefault("RESHARD_DIST_BACKEND", "gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    os.execvpe(sys.executable, cmd, env)


AUTO_EMULATED = None


def auto_emulate(args) -> None:
    """A world of more GPUs than the box shows (e.g. the scaling command run on a one-GPU box):
    instead of failing, run it emulated on cuda:0 (RESHARD_SAME_GPU; gloo plumbing when several
    processes share the device) and label the line (`emulated_on_one_gpu`, `emulation`)."""
    global DIST_BACKEND, AUTO_EMULATED
    if args.impl != "ours" or args.gpus <= 1 or os.environ.get("RESHARD_SAME_GPU"):
        return
    import torch

    n = torch.cuda.device_count()
    if n == 0 or n >= args.gpus:
        return
    os.environ["RESHARD_SAME_GPU"] = "1"
    if int(os.environ.get("WORLD_SIZE", "1")) > 1 or args.workload in DATASET:
        os.environ["RESHARD_DIST_BACKEND"] = "gloo"
        DIST_BACKEND = "gloo"
    AUTO_EMULATED = f"--gpus {args.gpus} on a box with {n} CUDA device(s): every world GPU emulated on cuda:0"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS) + sorted(DATASET))
    ap.add_argument("--tile-kib", type=int, default=256)
    ap.add_argument("--mode", choices=["distributed", "central"], default="distributed",
                    help="apply_plan mode (SPEC.md:466): central stages every moved fragment on GPU 0")
    ap.add_argument("--waves", type=int, default=0, help="catalog windows run one after another (0: automatic)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-p2p-probe", action="store_true")
    ap.add_argument("--no-digests", action="store_true", help="skip the ExecutionReport FNV digests (off the clock)")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    auto_emulate(args)
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.workload in DATASET:
        relaunch_under_torchrun(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
