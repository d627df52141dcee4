"""Generate the golden fixtures of this directory from the REFERENCE's own compiled code.

    python tests/golden/make_golden.py

tensor_core_kat.json: slice / merge / grid cells / grid_refine / even_split / Range::parse
    cases with inputs, outputs and error names, produced by oracle/_ref/libptc_ref.so, i.e. by
    /root/reference/proj/src/tensor/*.cpp compiled unmodified (plus the split_grid.hpp shim).
    The SPEC examples and the survey's derived KATs are included
    verbatim, followed by seeded random cases.
fig6_plan.txt: the Fig. 6 plan (acceptance #4) from the restated planner over
    the reference tensor-core.
plans.json: plan statistics of the BASELINE configurations.
Run in the build container (needs /root/reference); the outputs are committed.
"""
from __future__ import annotations

import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

from oracle.oracle import Oracle, OracleError  # noqa: E402

W = {0: 4, 1: 2, 2: 8, 3: 1}


def iota_bytes(dtype, shape):
    n = int(np.prod(shape)) if shape else 1
    if dtype == 0:
        return np.arange(n, dtype=np.float32).view(np.uint8)
    if dtype == 1:
        return np.arange(n, dtype=np.float16).view(np.uint8)
    if dtype == 2:
        return np.arange(n, dtype=np.int64).view(np.uint8)
    return (np.arange(n) % 251).astype(np.uint8)


def call(fn):
    try:
        out = fn()
        return {"ok": out}
    except OracleError as e:
        return {"error": e.name}


def main():
    ref = Oracle(reference=True)
    assert ref.uses_reference_core
    rng = random.Random(2312)
    kat = {"slice": [], "merge": [], "grid_cells": [], "grid_refine": [], "even_split": [], "parse": []}

    def add_slice(dtype, shape, box, payload=None):
        pay = iota_bytes(dtype, shape) if payload is None else payload
        r = call(lambda: ref.slice(dtype, shape, pay, box).tobytes().hex())
        kat["slice"].append({"dtype": dtype, "shape": list(shape), "payload": pay.tobytes().hex(),
                             "box": [list(x) for x in box], **r})

    # SPEC.md:60-62 and SURVEY §4
    add_slice(0, (4, 6), [(0, 4), (2, 4)])
    add_slice(0, (6,), [(2, 3)])
    add_slice(0, (4, 6), [(0, 4), (0, 6)])
    add_slice(0, (4, 6), [(0, 4), (2, 7)])      # RangeOutOfBounds
    add_slice(0, (4, 6), [(0, 4)])              # RankMismatch
    add_slice(0, (4, 6), [(2, 2), (0, 6)])      # empty interval
    for _ in range(150):
        rank = rng.randint(0, 4)
        shape = tuple(rng.randint(1, 7) for _ in range(rank))
        dtype = rng.choice([0, 1, 2, 3])
        box = []
        for e in shape:
            lo = rng.randint(0, e - 1)
            box.append((lo, rng.randint(lo + 1, e)))
        if rng.random() < 0.1 and box:
            i = rng.randrange(len(box))
            box[i] = (box[i][0], shape[i] + 1)
        add_slice(dtype, shape, box)

    def add_merge(parts, target):
        r = call(lambda: ref.merge(parts, target).tobytes().hex())
        kat["merge"].append({"parts": [{"box": [list(x) for x in b], "dtype": dt, "shape": list(sh),
                                        "payload": np.asarray(p, np.uint8).tobytes().hex()} for b, dt, sh, p in parts],
                             "target": list(target), **r})

    v6 = iota_bytes(0, (6,))
    add_merge([([(0, 3)], 0, (3,), v6[:12]), ([(3, 6)], 0, (3,), v6[12:])], (6,))
    add_merge([([(0, 1)], 0, (1,), v6[8:12]), ([(1, 2)], 0, (1,), v6[12:16])], (2,))
    add_merge([], (6,))                                                                  # TilingGap
    add_merge([([(0, 4)], 0, (4,), v6[:16]), ([(3, 6)], 0, (3,), v6[12:])], (6,))      # TilingOverlap
    add_merge([([(0, 3)], 0, (3,), v6[:12])], (6,))                                    # TilingGap
    add_merge([([(0, 3)], 0, (3,), v6[:12]), ([(3, 6)], 1, (3,), v6[:6])], (6,))       # DtypeMismatch
    add_merge([([(0, 3)], 0, (2,), v6[:8])], (6,))                                     # ShapeMismatch
    # SPEC.md:71 quadrants of a [4,6]
    q = iota_bytes(0, (4, 6))
    quads = [[(0, 2), (0, 3)], [(0, 2), (3, 6)], [(2, 4), (0, 3)], [(2, 4), (3, 6)]]
    add_merge([(b, 0, (2, 3), ref.slice(0, (4, 6), q, b)) for b in quads], (4, 6))
    for _ in range(100):
        rank = rng.randint(1, 3)
        shape = tuple(rng.randint(1, 6) for _ in range(rank))
        dtype = rng.choice([0, 1, 2, 3])
        pay = np.frombuffer(rng.randbytes(int(np.prod(shape)) * W[dtype]), np.uint8)
        pts = [sorted(rng.sample(range(1, e), rng.randint(0, min(2, e - 1)))) if e > 1 else [] for e in shape]
        cells = ref.grid_cells(shape, pts)
        parts = [(c, dtype, tuple(z - a for a, z in c), ref.slice(dtype, shape, pay, c)) for c in cells]
        rng.shuffle(parts)
        mode = rng.random()
        if mode < 0.1 and len(parts) > 1:
            parts = parts[1:]                                    # gap
        elif mode < 0.2 and len(parts) > 1:
            parts = parts + [parts[0]]                           # overlap
        add_merge(parts, shape)

    def add_grid(shape, pts):
        kat["grid_cells"].append({"shape": list(shape), "points": pts, **call(lambda: ref.grid_cells(shape, pts))})

    add_grid((6,), [[3]])
    add_grid((6,), [[2, 4]])
    add_grid((4, 6), [[], [3]])
    add_grid((5,), [[7]])            # InvalidSplitPoint
    add_grid((6,), [[3, 3]])         # InvalidSplitPoint (not strictly increasing)
    add_grid((6,), [[0]])
    add_grid((6, 2), [[3]])          # RankMismatch
    add_grid((), [])
    for _ in range(60):
        rank = rng.randint(1, 3)
        shape = tuple(rng.randint(1, 9) for _ in range(rank))
        pts = [sorted(rng.sample(range(1, e), rng.randint(0, min(3, e - 1)))) if e > 1 else [] for e in shape]
        add_grid(shape, pts)

    for a, b in [([[3]], [[2, 4]]), ([[3]], [[3]]), ([[]], [[1]]), ([[3]], [[1], [2]]), ([[1, 5], []], [[2], [3]])]:
        kat["grid_refine"].append({"a": a, "b": b, **call(lambda: ref.grid_refine(a, b))})
    for shape, dim, ways in [((6,), 0, 2), ((6,), 0, 3), ((6,), 0, 4), ((6,), 1, 2), ((6,), 0, 0), ((4, 8), 1, 4),
                             ((4, 8), 0, 1)]:
        kat["even_split"].append({"shape": list(shape), "dim": dim, "ways": ways,
                                  **call(lambda: ref.even_split(shape, dim, ways))})
    for text in ["[]", "[0:4,2:4]", "[2:3]", "[1:2,3:4,5:6]", "[ 1:2]", "[2:]", "[:2]", "1:2", "[1:2", "[1-2]",
                 "[1:2,]", "[,1:2]", "[18446744073709551615:1]", "[18446744073709551616:1]", "[+1:2]", "[3:1]"]:
        kat["parse"].append({"text": text, "spec": False, **call(lambda: ref.range_parse(text))})
    for text in ["[:,2:4]", "[:]", "[:,:]", "[1:2,:]", "[::]", "[]"]:
        kat["parse"].append({"text": text, "spec": True, **call(lambda: ref.range_parse(text, spec=True))})

    # SplitGrid::cell / cell_index_of, Range::offset_by, RangeSpec::resolve
    kat.update({"grid_cell": [], "cell_index_of": [], "offset_by": [], "spec_resolve": []})
    for shape, pts in [((6,), [[3]]), ((4, 6), [[], [3]]), ((4, 6), [[1, 3], [2]]), ((5,), [[7]]), ((), [])]:
        for index in range(8):
            kat["grid_cell"].append({"shape": list(shape), "points": pts, "index": index,
                                     **call(lambda: ref.grid_cell(shape, pts, index))})
    for _ in range(60):
        rank = rng.randint(1, 3)
        shape = tuple(rng.randint(1, 9) for _ in range(rank))
        pts = [sorted(rng.sample(range(1, e), rng.randint(0, min(3, e - 1)))) if e > 1 else [] for e in shape]
        box = []
        for e in shape:
            lo = rng.randint(0, e - 1)
            box.append((lo, rng.randint(lo + 1, e)))
        if rng.random() < 0.1:
            box[0] = (box[0][0], shape[0] + 1)
        kat["cell_index_of"].append({"shape": list(shape), "points": pts, "box": [list(x) for x in box],
                                     **call(lambda: ref.grid_cell_index_of(shape, pts, box))})
        index = rng.randint(0, 12)
        kat["grid_cell"].append({"shape": list(shape), "points": pts, "index": index,
                                 **call(lambda: ref.grid_cell(shape, pts, index))})
        outer = [(rng.randint(0, 4), 0) for _ in range(rank)]
        outer = [(a, a + rng.randint(1, 6)) for a, _ in outer]
        inner = []
        for a, z in outer:
            lo = rng.randint(0, z - a)
            inner.append((lo, lo + rng.randint(0, z - a - lo + 1)))
        if rng.random() < 0.1:
            outer = outer[:-1]
        kat["offset_by"].append({"box": [list(x) for x in inner], "outer": [list(x) for x in outer],
                                 **call(lambda: ref.offset_by(inner, outer))})
    for text, shape in [("[:,2:4]", (4, 6)), ("[:]", (5,)), ("[1:2,:]", (3, 3)), ("[:,2:7]", (4, 6)),
                        ("[:]", (4, 6)), ("[]", ()), ("[2:2]", (4,)), ("[0:4,0:6]", (4, 6))]:
        spec = ref.range_parse(text, spec=True)
        kat["spec_resolve"].append({"text": text, "shape": list(shape),
                                    **call(lambda: ref.spec_resolve(spec, shape))})

    with open(os.path.join(HERE, "tensor_core_kat.json"), "w") as f:
        json.dump(kat, f, indent=0, sort_keys=True)

    # Fig. 6 golden plan (acceptance #4)
    cat = ref.catalog([("t1", 0, (6,), 0, 0), ("t2", 0, (6,), 0, 1)])
    a = cat.build_strategy([(0, 0), (0, 1)], 2, 1, 1)
    b = cat.build_strategy([(0, i) for i in range(6)], 3, 2, 1)
    with open(os.path.join(HERE, "fig6_plan.txt"), "w") as f:
        f.write(a.plan(b).text())

    # plan statistics of the BASELINE configurations
    plans = {}
    devs = lambda n: [(0, i) for i in range(n)]  # noqa: E731
    specs = {
        "gpt2-small-tp2-to-pp2": ((768, 12, 1024, 50304, 0), (2, 1, 1, devs(2)), (1, 2, 1, devs(2)), []),
        "gpt3-1.3b-dp-scaleout": ((2048, 24, 2048, 50304, 1), (2, 1, 1, devs(2)), (2, 1, 2, devs(4)), []),
        "gpt3-6.7b-tp4pp2-to-tp2pp2dp2": ((4096, 32, 2048, 50304, 1), (4, 2, 1, devs(8)), (2, 2, 2, devs(8)), []),
        "gpt3-6.7b-recovery": ((4096, 32, 2048, 50304, 1), (2, 2, 2, devs(8)), (2, 2, 1, [(0, 0), (0, 2), (0, 5), (0, 7)]),
                               [(0, 1), (0, 3), (0, 4), (0, 6)]),
    }
    for name, ((h, L, S, V, k), (T1, P1, D1, d1), (T2, P2, D2, d2), failed) in specs.items():
        c = ref.catalog_gpt(h, L, S, V, k)
        p = c.build_strategy(d1, T1, P1, D1).plan(c.build_strategy(d2, T2, P2, D2), failed=failed)
        cost = p.cost()
        plans[name] = {**p.stats(), "max_ingress": max(v[0] for v in cost.values()),
                       "max_egress": max(v[1] for v in cost.values()),
                       "text_fnv1a64": ref.fnv1a64(p.text().encode())}
    with open(os.path.join(HERE, "plans.json"), "w") as f:
        json.dump(plans, f, indent=1, sort_keys=True)
    print("wrote", os.listdir(HERE))


if __name__ == "__main__":
    main()
