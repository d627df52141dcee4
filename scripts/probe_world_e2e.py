#!/usr/bin/env python
"""A/B of the two host-buffer paths on ONE GPU (GPT-3 1.3B DP scale-out): rs_executor_run_host
(64 destination-ordered chunks, one upload and one download stream) vs
rs_executor_run_host_world (pipelined rounds, the multi-GPU path) with a one-GPU world, so the
world pipeline's own efficiency is measured without several world GPUs sharing one PCIe link."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2312_05181_b200 as rs  # noqa: E402


def main():
    cat, a, b, plan, sg, dg = bench.build_plan(rs, "gpt3-1.3b-dp-scaleout", 1)
    ctx = rs.Context(1, [0], [0])
    ex = rs.Executor(ctx, plan, sg, dg)
    ex.allocate_local()
    ex.prepare()
    ex.fill_sources()
    s_b, d_b = ex.arena_bytes(0)
    hs, hd = rs.host_alloc(s_b), rs.host_alloc(d_b)
    ctx.dtoh(0, hs, ex.arenas[0][0], s_b)
    out = {}
    ex.run_host(0, hs, hd)
    out["run_host_ms"] = [round(ex.run_host(0, hs, hd)["ms"], 1) for _ in range(3)]
    for pl in ("1", "0"):
        os.environ["RESHARD_WORLD_PIPELINE"] = pl
        ex.run_host_world([hs], [hd])
        out[f"run_host_world_pipeline{pl}_ms"] = [round(ex.run_host_world([hs], [hd]), 1) for _ in range(3)]
    out["verify"] = ex.verify()
    out["bytes"] = {"h2d": s_b, "d2h": d_b}
    print(json.dumps(out))
    rs.host_free(hs)
    rs.host_free(hd)


if __name__ == "__main__":
    main()
