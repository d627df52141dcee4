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


@pytest.mark.parametrize("kernel", ["bulk_strided", "bulk", "ldg", "bulk_strided-peer"])
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
    assert line["e2e"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0  # multi-rank host-buffer path ran
    assert line["fabric"]["t_roof_ms"] > 0 and line["fabric"]["bottleneck"]["term"] in ("hbm", "nvlink_in", "nvlink_out")


def test_two_ranks_dataset_repartition():
    """configs[4] through torchrun with 2 ranks sharing cuda:0: new DP rank d of each event
    runs on GPU d % 2, the line aggregates every rank's samples (10^8 x 1.04) and each
    rank's spot check of positions / entries against the host restatement passes."""
    env = dict(os.environ, RESHARD_DIST_BACKEND="gloo", RESHARD_SAME_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--workload", "dataset-100m-dp2to4to8", "--no-cpu-baseline", "--no-e2e"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    line = json.loads([x for x in p.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["samples_per_step"] == 104_000_000
    assert line["spot_check"] == {"pos": True, "ent": True}
    assert line["shuffle_epoch_gpu"]["bit_identical_to_host"]
