#!/usr/bin/env python
"""Checkpoint I/O throughput on the GPU box: save the GPT-2 small and GPT-3
1.3B source layouts as PTX1 files (D2H through double-buffered pinned staging + file writes)
into a RAM-backed directory (/dev/shm, so the number is the staging path, not a disk), load
them back, verify every destination byte after a reshard from the loaded state."""
import json
import os
import shutil
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2312_05181_b200 as rs  # noqa: E402
from paper_2312_05181_b200 import checkpoint as ck  # noqa: E402

ctx = rs.Context(1, [0], [0])
base = "/dev/shm" if os.path.isdir("/dev/shm") else None
for name, (h, L, S, V, kind), (T1, P1, D1), (T2, P2, D2) in [
        ("gpt2-small", (768, 12, 1024, 50304, rs.FP32_ADAM), (2, 1, 1), (1, 2, 1)),
        ("gpt3-1.3b", (2048, 24, 2048, 50304, rs.MIXED_ADAM), (2, 1, 1), (2, 1, 2))]:
    cat = rs.Catalog.gpt(h, L, S, V, kind)
    a = cat.build_strategy([(0, i) for i in range(T1 * P1 * D1)], T1, P1, D1)
    b = cat.build_strategy([(0, i) for i in range(T2 * P2 * D2)], T2, P2, D2)
    ex = rs.Executor(ctx, rs.generate_plan(a, b), [0] * (T1 * P1 * D1), [0] * (T2 * P2 * D2))
    ex.allocate_local()
    ex.prepare()
    ex.fill_sources()
    d = tempfile.mkdtemp(dir=base)
    try:
        sv = ck.checkpoint_save(ex, d, 0)
        ex2 = rs.Executor(ctx, rs.generate_plan(a, b), [0] * (T1 * P1 * D1), [0] * (T2 * P2 * D2))
        ex2.allocate_local()
        ex2.prepare()
        ld = ck.checkpoint_load(ex2, d)
        ex2.apply()
        bad = ex2.verify()
    finally:
        shutil.rmtree(d, ignore_errors=True)
    print(json.dumps({"model": name, "dir": base or "tmp", "files": sv["files"], "gb": round(sv["bytes"] / 1e9, 3),
                      "save_gbs": round(sv["bytes"] / sv["seconds"] / 1e9, 2),
                      "load_gbs": round(ld["bytes"] / ld["seconds"] / 1e9, 2), "mismatched_bytes": bad}), flush=True)
