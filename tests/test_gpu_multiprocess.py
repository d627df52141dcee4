"""The one-process-per-GPU path end to end on the single available GPU: two torchrun ranks
share cuda:0, exchange CUDA-IPC handles of their destination arenas, and push their
fragments into each other's arenas (K1/K2/K3 kernels writing through IPC mappings).
Correctness only (both ranks compete for one GPU): every destination byte must verify."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("kernel", ["bulk_strided", "bulk", "ldg", "bulk_strided-peer", "bulk_dyn"])
def test_two_ranks_one_gpu_ipc_push(kernel):
    env = dict(os.environ, RESHARD_DIST_BACKEND="gloo", RESHARD_SAME_GPU="1", RESHARD_COPY_KERNEL=kernel.split("-")[0])
    if kernel.endswith("-peer"):  # TMA bulk stores through the IPC mapping as well
        env["RESHARD_BULK_PEER"] = "1"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--workload", "gpt2-small-tp2-to-pp2", "--no-cpu-baseline", "--e2e-steps", "1"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    line = json.loads([x for x in p.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["verify_mismatched_bytes"] == 0
    # world time from rank 0's start to the last rank's interprocess "done" event
    assert "interprocess" in line["timing"] and line["value"] >= 0.99 * line["ms_max_gpu_kernel"] > 0
    assert line["e2e"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0  # multi-rank host-buffer path ran
    # both host-buffer forms ran: per-rank phases and rank 0's single-process world API
    assert "world_api" in line["e2e"] or "per_rank_phases" in line["e2e"]
    world = line["e2e"].get("world_api", line["e2e"])
    assert world["mismatched_bytes"] == 0 and "run_host_world" in world["path"]
    assert line["fabric"]["t_roof_ms"] > 0 and line["fabric"]["bottleneck"]["term"] in ("hbm", "nvlink_in", "nvlink_out")


def test_two_ranks_dataset_repartition():
    """configs[4] with --gpus 2 and NO launcher: bench.py re-executes itself under torchrun
    (2 ranks sharing cuda:0, gloo): new DP rank d of each event runs on GPU d % 2, the line
    aggregates every rank's samples (10^8 x 1.04) and each rank's spot check of positions /
    entries against the host restatement passes."""
    env = dict(os.environ, RESHARD_SAME_GPU="1")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--workload", "dataset-100m-dp2to4to8", "--no-cpu-baseline", "--no-e2e"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    line = json.loads([x for x in p.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["samples_per_step"] == 104_000_000
    assert line["spot_check"] == {"pos": True, "ent": True}
    assert line["shuffle_epoch_gpu"]["bit_identical_to_host"]


def _bench_no_launcher(n, workload, *extra, timeout=1200):
    env = dict(os.environ, RESHARD_SAME_GPU="1")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    cmd = [sys.executable, "bench.py", "--gpus", str(n), "--steps", "3", "--warmup", "3", "--workload", workload,
           "--no-cpu-baseline", "--e2e-steps", "1", *extra]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, p.stderr[-3000:]
    return json.loads([x for x in p.stdout.splitlines() if x.startswith("{")][-1])


@pytest.mark.parametrize("n", [2, 8])
def test_single_process_world_no_launcher(n):
    """`python bench.py --gpus N` with no launcher drives an N-GPU world from one
    process (here every world GPU emulated on cuda:0): one common start event, every GPU's
    kernels, the last GPU's end; the host-buffer path through rs_executor_run_host_world; every
    destination byte verifies (GPUs 2..7 of the 8-GPU world host nothing: empty arenas)."""
    line = _bench_no_launcher(n, "gpt2-small-tp2-to-pp2")
    assert line["n_gpus"] == n and line["verify_mismatched_bytes"] == 0 and line["emulated_on_one_gpu"]
    assert line["config"]["n_gpus"] == n and line["gpu_launches"] > 0
    assert line["e2e"]["value"] > 0 and line["e2e"]["mismatched_bytes"] == 0
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and "run_host_world" in line["e2e"]["path"]
    assert line["value"] >= line["ms_max_gpu_kernel"] * 0.999  # the world time contains every GPU's kernels
    assert line["fabric"]["t_roof_ms"] > 0 and line["roofline"]["bound"] == "hbm"


def test_single_process_world_scaleout_full_size():
    """BASELINE configs[1] at full size as the driver's N=4 scaling run launches it (no
    launcher), emulated on one GPU: GPT-3 1.3B (TP2,PP1,DP1)->(TP2,PP1,DP2), 18.5 GB moved,
    every destination byte verified (K7), the host-buffer path included."""
    line = _bench_no_launcher(4, "gpt3-1.3b-dp-scaleout")
    assert line["verify_mismatched_bytes"] == 0 and line["moved_bytes"] == 18_484_379_648
    assert line["e2e"]["mismatched_bytes"] == 0
    assert line["fabric"]["max_egress_gb"] > 9


def test_elastic_sequence_process_and_in_process_agree():
    """SPEC acceptance #10: the §6.2 sequence (2,4,2) -> (2,4,1) -> (2,2,1) (and back) on a toy
    model, each step reading what the previous one wrote, gives identical plans, byte counts and
    per-cell digests with one process driving a 4-GPU world and with one process per GPU (4
    torchrun ranks, CUDA-IPC arenas); every destination byte of every step verifies."""
    env = dict(os.environ, RESHARD_SAME_GPU="1")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    runs = {}
    p = subprocess.run([sys.executable, "scripts/elastic_sequence.py", "--world", "4"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    runs["in-process"] = json.loads([x for x in p.stdout.splitlines() if x.startswith("{")][-1])
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=4", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), "scripts/elastic_sequence.py", "--world", "4"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    runs["process"] = json.loads([x for x in p.stdout.splitlines() if x.startswith("{")][-1])
    a, b = runs["in-process"], runs["process"]
    assert a["mode"] == "in-process" and b["mode"] == "process"
    assert len(a["steps"]) == 3
    for sa, sb in zip(a["steps"], b["steps"]):
        assert sa["mismatched_bytes"] == 0 and sb["mismatched_bytes"] == 0
        assert sa["executed_bytes"] == sa["moved_bytes"] + sa["relayout_bytes"]
        assert len(sa["digests"]) > 0
    # DP 2 -> 1 keeps the first replica in place (nothing moves); PP 4 -> 2 re-stages; the way
    # back re-stages and fans out to a second replica
    assert a["steps"][0]["moved_bytes"] == 0 and a["steps"][1]["moved_bytes"] > 0 and a["steps"][2]["moved_bytes"] > 0
    assert a["steps"] == b["steps"]


def test_more_gpus_than_the_box_runs_emulated_and_labelled():
    """The driver's scaling command on a box with fewer GPUs (no RESHARD_SAME_GPU set): the world
    runs emulated on cuda:0 and the line says so, instead of failing."""
    import torch

    if torch.cuda.device_count() >= 2:
        pytest.skip("the box has 2 GPUs")
    env = dict(os.environ)
    for k in ("RESHARD_SAME_GPU", "WORLD_SIZE", "RANK", "LOCAL_RANK", "RESHARD_DIST_BACKEND"):
        env.pop(k, None)
    p = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3", "--workload",
                        "gpt2-small-tp2-to-pp2", "--no-cpu-baseline", "--no-e2e", "--no-digests"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    line = json.loads([x for x in p.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["emulated_on_one_gpu"] is True and "emulated" in line["emulation"]
    assert line["verify_mismatched_bytes"] == 0
