"""ctypes front-end of the CPU oracle — TEST INFRASTRUCTURE ONLY.

Loads either ``oracle/liboracle.so`` (the restatement, oracle.cpp) or
``oracle/_ref/libptc_ref.so`` (the same restated upper layers over the reference's own
compiled tensor-core, /root/reference/proj/src/tensor/*.cpp).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl reference`` legs may
import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
MAXR = 8
ERRC = [
    "RangeOutOfBounds", "RankMismatch", "ShapeMismatch", "TilingGap", "TilingOverlap",
    "DtypeMismatch", "InvalidSplitPoint", "InvalidTensor", "IndivisibleLayerCount",
    "IndivisibleSliceDim", "DeviceCountMismatch", "InvalidJobConfig", "MalformedConfig",
    "InconsistentBaseShape", "CoverageGap", "UnknownDevice", "CatalogMismatch",
    "UnsatisfiableFragment", "NoSource", "NotFound", "IndivisibleBatch", "StepBeyondEpoch",
    "IndexOutOfRange", "InvalidReplicaCount", "MalformedFrame", "UnknownVerb", "BadRange",
    "ConnectionFailed", "CheckpointRequired", "LayoutMismatch", "IoError", "ScriptError",
    "Internal",
]
WIDTH = {0: 4, 1: 2, 2: 8, 3: 1}
LAYER_PRE, LAYER_POST = -1, -2

u8p = np.ctypeslib.ndpointer(np.uint8, flags="C")


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code
        self.name = ERRC[code] if 0 <= code < len(ERRC) else "Unknown"


def lib_path(reference: bool = False) -> str:
    return os.path.join(HERE, "_ref", "libptc_ref.so") if reference else os.path.join(HERE, "liboracle.so")


def build(reference: bool | None = None) -> None:
    """Compile the restatement (always) and the reference-core variant when the
    reference sources are present (this container; the GPU box uses prebuilt files)."""
    targets = ["all"]
    ref_root = os.environ.get("REF_ROOT", "/root/reference/proj")
    if reference or (reference is None and os.path.isdir(ref_root)):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, f"REF_ROOT={ref_root}", *targets], check=True)


def _box_arrays(boxes):
    n = len(boxes)
    lo = np.zeros((max(n, 1), MAXR), np.uint64)
    hi = np.zeros((max(n, 1), MAXR), np.uint64)
    for i, b in enumerate(boxes):
        for d, (a, z) in enumerate(b):
            lo[i, d], hi[i, d] = a, z
    return lo, hi


class Oracle:
    def __init__(self, reference: bool = False, path: str | None = None):
        path = path or lib_path(reference)
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library not built: {path}")
        self.path = path
        L = self.lib = C.CDLL(path)
        L.orc_last_error.restype = C.c_char_p
        L.orc_errc_name.restype = C.c_char_p
        L.orc_fnv1a64.restype = C.c_uint64
        L.orc_fnv1a64.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_splitmix64_next.restype = C.c_uint64
        L.orc_splitmix64_next.argtypes = [C.POINTER(C.c_uint64)]
        L.orc_next_below.restype = C.c_uint64
        L.orc_next_below.argtypes = [C.POINTER(C.c_uint64), C.c_uint64]
        L.orc_stream_bytes.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, u8p]
        L.orc_path_seed.restype = C.c_uint64
        L.orc_path_seed.argtypes = [C.c_char_p]
        L.orc_catalog_new.restype = C.c_void_p
        L.orc_catalog_gpt.restype = C.c_void_p
        L.orc_catalog_gpt.argtypes = [C.c_uint64] * 4 + [C.c_int]
        for fn in ("orc_catalog_free", "orc_ptc_free", "orc_plan_free", "orc_state_free"):
            getattr(L, fn).argtypes = [C.c_void_p]
        L.orc_catalog_size.argtypes = [C.c_void_p]
        L.orc_plan_text.restype = C.c_int64
        L.orc_plan_text.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
        self.uses_reference_core = bool(L.orc_uses_reference_core())

    # ---- plumbing ----
    def _chk(self, rc: int):
        if rc != 0:
            raise OracleError(rc - 1, self.lib.orc_last_error().decode())

    # ---- tensor core ----
    def slice(self, dtype: int, shape, payload, box):
        """reference slice(t, r) (tensor.cpp:61-78) on a host payload."""
        sh = np.zeros(MAXR, np.uint64)
        sh[: len(shape)] = shape
        lo, hi = _box_arrays([box])
        n = 1
        for a, z in box:
            n *= max(int(z) - int(a), 0)
        w = WIDTH.get(dtype, 1)
        out = np.zeros(max(n * w, 1), np.uint8)
        pay = np.ascontiguousarray(payload, dtype=np.uint8)
        self._chk(self.lib.orc_slice(C.c_int(dtype), C.c_int(len(shape)), sh.ctypes.data_as(C.c_void_p),
                                     pay.ctypes.data_as(C.c_void_p), C.c_int(len(box)),
                                     lo.ctypes.data_as(C.c_void_p), hi.ctypes.data_as(C.c_void_p),
                                     out.ctypes.data_as(C.c_void_p)))
        return out[: n * w]

    def merge(self, parts, target_shape):
        """parts: list of (box, dtype, shape, payload)."""
        n = len(parts)
        dt = np.array([p[1] for p in parts] or [0], np.int32)
        rk = np.array([len(p[2]) for p in parts] or [0], np.int32)
        rr = np.array([len(p[0]) for p in parts] or [0], np.int32)
        shapes = np.zeros((max(n, 1), MAXR), np.uint64)
        for i, p in enumerate(parts):
            shapes[i, : len(p[2])] = p[2]
        lo, hi = _box_arrays([p[0] for p in parts])
        pays = [np.ascontiguousarray(p[3], dtype=np.uint8) for p in parts]
        ptrs = (C.c_void_p * max(n, 1))(*[x.ctypes.data for x in pays])
        ts = np.zeros(MAXR, np.uint64)
        ts[: len(target_shape)] = target_shape
        tot = 1
        for e in target_shape:
            tot *= int(e)
        w = WIDTH.get(parts[0][1], 1) if parts else 1
        out = np.zeros(max(tot * w, 1), np.uint8)
        self._chk(self.lib.orc_merge(C.c_int(n), dt.ctypes.data_as(C.c_void_p), rk.ctypes.data_as(C.c_void_p),
                                     shapes.ctypes.data_as(C.c_void_p), ptrs, rr.ctypes.data_as(C.c_void_p),
                                     lo.ctypes.data_as(C.c_void_p), hi.ctypes.data_as(C.c_void_p),
                                     C.c_int(len(target_shape)), ts.ctypes.data_as(C.c_void_p),
                                     out.ctypes.data_as(C.c_void_p)))
        return out[: tot * w]

    def grid_cells(self, shape, points):
        rank = len(shape)
        sh = np.array(list(shape) + [0], np.uint64)
        npts = np.array([len(p) for p in points] + [0], np.int32)
        pts = np.array([x for p in points for x in p] + [0], np.uint64)
        cap = 4096
        lo = np.zeros((cap, MAXR), np.uint64)
        hi = np.zeros((cap, MAXR), np.uint64)
        n = C.c_int(0)
        self._chk(self.lib.orc_grid_cells(C.c_int(rank), sh.ctypes.data_as(C.c_void_p),
                                          npts.ctypes.data_as(C.c_void_p), pts.ctypes.data_as(C.c_void_p),
                                          C.c_int(cap), lo.ctypes.data_as(C.c_void_p), hi.ctypes.data_as(C.c_void_p),
                                          C.byref(n)))
        return [[(int(lo[i, d]), int(hi[i, d])) for d in range(rank)] for i in range(n.value)]

    def grid_refine(self, a, b):
        na = np.array([len(p) for p in a] + [0], np.int32)
        pa = np.array([x for p in a for x in p] + [0], np.uint64)
        nb = np.array([len(p) for p in b] + [0], np.int32)
        pb = np.array([x for p in b for x in p] + [0], np.uint64)
        nout = np.zeros(max(len(a), 1), np.int32)
        pout = np.zeros(len(pa) + len(pb) + 1, np.uint64)
        self._chk(self.lib.orc_grid_refine(C.c_int(len(a)), na.ctypes.data_as(C.c_void_p),
                                           pa.ctypes.data_as(C.c_void_p), C.c_int(len(b)),
                                           nb.ctypes.data_as(C.c_void_p), pb.ctypes.data_as(C.c_void_p),
                                           nout.ctypes.data_as(C.c_void_p), pout.ctypes.data_as(C.c_void_p)))
        res, k = [], 0
        for d in range(len(a)):
            res.append([int(x) for x in pout[k : k + nout[d]]])
            k += nout[d]
        return res

    def even_split(self, shape, dim, ways):
        sh = np.array(list(shape) + [0], np.uint64)
        nout = np.zeros(max(len(shape), 1), np.int32)
        pout = np.zeros(max(int(ways), 1) + 1, np.uint64)
        self._chk(self.lib.orc_even_split(C.c_int(len(shape)), sh.ctypes.data_as(C.c_void_p), C.c_int(dim),
                                          C.c_uint64(ways), nout.ctypes.data_as(C.c_void_p),
                                          pout.ctypes.data_as(C.c_void_p)))
        res, k = [], 0
        for d in range(len(shape)):
            res.append([int(x) for x in pout[k : k + nout[d]]])
            k += nout[d]
        return res

    def range_parse(self, text: str, spec: bool = False):
        rank = C.c_int(0)
        lo = np.zeros(MAXR, np.uint64)
        hi = np.zeros(MAXR, np.uint64)
        self._chk(self.lib.orc_range_parse(text.encode(), C.c_int(int(spec)), C.byref(rank),
                                           lo.ctypes.data_as(C.c_void_p), hi.ctypes.data_as(C.c_void_p)))
        M = (1 << 64) - 1
        return [None if (spec and int(lo[i]) == M and int(hi[i]) == M) else (int(lo[i]), int(hi[i]))
                for i in range(rank.value)]

    # ---- hash / rng ----
    def fnv1a64(self, data: bytes | np.ndarray) -> int:
        a = np.frombuffer(bytes(data), np.uint8) if not isinstance(data, np.ndarray) else np.ascontiguousarray(data, np.uint8)
        return int(self.lib.orc_fnv1a64(a.ctypes.data_as(C.c_void_p) if a.size else None, a.size))

    def splitmix64(self, state: int, n: int):
        s = C.c_uint64(state)
        return [int(self.lib.orc_splitmix64_next(C.byref(s))) for _ in range(n)], s.value

    def next_below(self, state: int, n: int):
        s = C.c_uint64(state)
        v = int(self.lib.orc_next_below(C.byref(s), C.c_uint64(n)))
        return v, s.value

    def stream_bytes(self, seed: int, off: int, n: int) -> np.ndarray:
        out = np.zeros(max(n, 1), np.uint8)
        self.lib.orc_stream_bytes(C.c_uint64(seed), C.c_uint64(off), C.c_uint64(n), out)
        return out[:n]

    def path_seed(self, path: str) -> int:
        return int(self.lib.orc_path_seed(path.encode()))

    # ---- catalog / PTC / plan / apply ----
    def catalog_gpt(self, h, L, S, V, kind) -> "Catalog":
        return Catalog(self, self.lib.orc_catalog_gpt(h, L, S, V, kind))

    def catalog(self, entries) -> "Catalog":
        """entries: list of (path, dtype, shape, tp_dim, layer)."""
        c = Catalog(self, self.lib.orc_catalog_new())
        for path, dtype, shape, tp, layer in entries:
            sh = np.array(list(shape) + [0], np.uint64)
            self._chk(self.lib.orc_catalog_add(C.c_void_p(c.h), path.encode(), C.c_int(dtype), C.c_int(len(shape)),
                                               sh.ctypes.data_as(C.c_void_p), C.c_int(tp), C.c_int(layer)))
        return c

    # ---- dataset ----
    def shuffle_epoch(self, n: int, seed: int, epoch: int) -> np.ndarray:
        out = np.zeros(max(n, 1), np.uint64)
        self.lib.orc_shuffle_epoch(C.c_uint64(n), C.c_uint64(seed), C.c_uint64(epoch), out.ctypes.data_as(C.c_void_p))
        return out[:n]

    def repartition_counts(self, n, B, at_step, dp):
        out = np.zeros(max(dp, 1), np.uint64)
        self._chk(self.lib.orc_repartition_counts(C.c_uint64(n), C.c_uint64(B), C.c_uint64(at_step),
                                                  C.c_uint64(dp), out.ctypes.data_as(C.c_void_p)))
        return [int(x) for x in out[:dp]]

    def repartition_positions(self, n, B, at_step, dp, d):
        cnt = self.repartition_counts(n, B, at_step, dp)[d] if d < dp else 0
        out = np.zeros(max(cnt, 1), np.uint64)
        self._chk(self.lib.orc_repartition_positions(C.c_uint64(n), C.c_uint64(B), C.c_uint64(at_step),
                                                     C.c_uint64(dp), C.c_uint64(d), out.ctypes.data_as(C.c_void_p)))
        return out[:cnt]

    def locate_sample(self, n, B, at_step, dp, d, k, perm, samples, file_class):
        out = np.zeros(4, np.uint64)
        self._chk(self.lib.orc_locate_sample(
            C.c_uint64(n), C.c_uint64(B), C.c_uint64(at_step), C.c_uint64(dp), C.c_uint64(d), C.c_uint64(k),
            np.ascontiguousarray(perm, np.uint64).ctypes.data_as(C.c_void_p),
            np.ascontiguousarray(samples, np.uint64).ctypes.data_as(C.c_void_p),
            np.ascontiguousarray(file_class, np.uint8).ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p)))
        return tuple(int(x) for x in out)

    def dataset_gather(self, n, B, at_step, dp, d, perm, samples, file_class, n_threads=1):
        cnt = self.repartition_counts(n, B, at_step, dp)[d]
        # outputs written once here, before the timed call: np.zeros maps pages lazily and the
        # first-touch page faults (257-674 ms across boxes for config 5) would be timed as gather work
        pos = np.empty(max(cnt, 1), np.uint64)
        ent = np.empty((max(cnt, 1), 3), np.uint64)
        boff = np.empty(max(cnt, 1), np.uint64)
        qidx = np.empty(max(cnt, 1), np.uint32)
        for a in (pos, ent, boff, qidx):
            a.fill(0)
        qcount = np.zeros(3, np.uint64)
        secs = C.c_double(0)
        self._chk(self.lib.orc_dataset_gather(
            C.c_uint64(n), C.c_uint64(B), C.c_uint64(at_step), C.c_uint64(dp), C.c_uint64(d),
            perm.ctypes.data_as(C.c_void_p), samples.ctypes.data_as(C.c_void_p),
            file_class.ctypes.data_as(C.c_void_p), pos.ctypes.data_as(C.c_void_p), ent.ctypes.data_as(C.c_void_p),
            boff.ctypes.data_as(C.c_void_p), qidx.ctypes.data_as(C.c_void_p), qcount.ctypes.data_as(C.c_void_p),
            C.c_int(n_threads), C.byref(secs)))
        return dict(pos=pos[:cnt], ent=ent[:cnt], boff=boff[:cnt], qidx=qidx[:cnt],
                    qcount=[int(x) for x in qcount], seconds=secs.value)


class _Handle:
    _free = ""

    def __init__(self, o: Oracle, h):
        self.o, self.h = o, h

    def __del__(self):
        if getattr(self, "h", None):
            getattr(self.o.lib, self._free)(C.c_void_p(self.h))
            self.h = None


class Catalog(_Handle):
    _free = "orc_catalog_free"

    def __len__(self):
        return self.o.lib.orc_catalog_size(C.c_void_p(self.h))

    def entry(self, i):
        name = C.create_string_buffer(256)
        dt, rk, tp, ly = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        sh = np.zeros(MAXR, np.uint64)
        self.o._chk(self.o.lib.orc_catalog_get(C.c_void_p(self.h), C.c_int(i), name, C.c_int(256), C.byref(dt),
                                               C.byref(rk), sh.ctypes.data_as(C.c_void_p), C.byref(tp), C.byref(ly)))
        return (name.value.decode(), dt.value, tuple(int(x) for x in sh[: rk.value]), tp.value, ly.value)

    def entries(self):
        return [self.entry(i) for i in range(len(self))]

    def build_strategy(self, devices, T, P, D) -> "Ptc":
        w = np.array([d[0] for d in devices] + [0], np.uint32)
        l = np.array([d[1] for d in devices] + [0], np.uint32)
        out = C.c_void_p()
        self.o._chk(self.o.lib.orc_build_strategy(C.c_void_p(self.h), C.c_int(len(devices)),
                                                  w.ctypes.data_as(C.c_void_p), l.ctypes.data_as(C.c_void_p),
                                                  C.c_int(T), C.c_int(P), C.c_int(D), C.byref(out)))
        return Ptc(self.o, out.value, self)

    def base_bytes(self, t):
        _, dt, shape, _, _ = self.entry(t)
        n = WIDTH[dt]
        for e in shape:
            n *= e
        out = np.zeros(max(n, 1), np.uint8)
        self.o._chk(self.o.lib.orc_base_bytes(C.c_void_p(self.h), C.c_int(t), out.ctypes.data_as(C.c_void_p)))
        return out[:n]

    def box_bytes(self, t, box):
        _, dt, shape, _, _ = self.entry(t)
        n = WIDTH[dt]
        for a, z in box:
            n *= z - a
        lo, hi = _box_arrays([box])
        out = np.zeros(max(n, 1), np.uint8)
        self.o._chk(self.o.lib.orc_box_bytes(C.c_void_p(self.h), C.c_int(t), C.c_int(len(box)),
                                             lo.ctypes.data_as(C.c_void_p), hi.ctypes.data_as(C.c_void_p),
                                             out.ctypes.data_as(C.c_void_p)))
        return out[:n]

    def base_digest(self, t):
        d = C.c_uint64()
        self.o._chk(self.o.lib.orc_base_digest(C.c_void_p(self.h), C.c_int(t), C.byref(d)))
        return d.value


class Ptc(_Handle):
    _free = "orc_ptc_free"

    def __init__(self, o, h, cat):
        super().__init__(o, h)
        self.cat = cat

    def validate(self):
        buf = C.create_string_buffer(1 << 16)
        n = C.c_int()
        self.o._chk(self.o.lib.orc_validate(C.c_void_p(self.h), buf, C.c_int(1 << 16), C.byref(n)))
        return [x for x in buf.value.decode().split("\n") if x]

    def set_alpha(self, part, devices):
        w = np.array([d[0] for d in devices] + [0], np.uint32)
        l = np.array([d[1] for d in devices] + [0], np.uint32)
        self.o._chk(self.o.lib.orc_ptc_set_alpha(C.c_void_p(self.h), C.c_int(part), C.c_int(len(devices)),
                                                 w.ctypes.data_as(C.c_void_p), l.ctypes.data_as(C.c_void_p)))

    def set_sigma(self, t, points):
        npts = np.array([len(p) for p in points] + [0], np.int32)
        pts = np.array([x for p in points for x in p] + [0], np.uint64)
        self.o._chk(self.o.lib.orc_ptc_set_sigma(C.c_void_p(self.h), C.c_int(t), C.c_int(len(points)),
                                                 npts.ctypes.data_as(C.c_void_p), pts.ctypes.data_as(C.c_void_p)))

    def hosted(self, dev):
        cap = 1 << 16
        t = np.zeros(cap, np.int32)
        lo = np.zeros((cap, MAXR), np.uint64)
        hi = np.zeros((cap, MAXR), np.uint64)
        n = C.c_int()
        self.o._chk(self.o.lib.orc_hosted(C.c_void_p(self.h), C.c_uint32(dev[0]), C.c_uint32(dev[1]), C.c_int(cap),
                                          t.ctypes.data_as(C.c_void_p), lo.ctypes.data_as(C.c_void_p),
                                          hi.ctypes.data_as(C.c_void_p), C.byref(n)))
        res = []
        for i in range(n.value):
            ti = int(t[i])
            r = len(self._shape(ti))
            res.append((ti, [(int(lo[i, d]), int(hi[i, d])) for d in range(r)]))
        return res

    def _shape(self, t):
        if not hasattr(self, "_shapes"):
            self._shapes = {}
        if t not in self._shapes:
            self._shapes[t] = self.cat.entry(t)[2]
        return self._shapes[t]

    def plan(self, other: "Ptc", failed=()) -> "Plan":
        fw = np.array([d[0] for d in failed] + [0], np.uint32)
        fl = np.array([d[1] for d in failed] + [0], np.uint32)
        out = C.c_void_p()
        self.o._chk(self.o.lib.orc_generate_plan(C.c_void_p(self.h), C.c_void_p(other.h), C.c_int(len(failed)),
                                                 fw.ctypes.data_as(C.c_void_p), fl.ctypes.data_as(C.c_void_p),
                                                 C.byref(out)))
        return Plan(self.o, out.value, self, other)

    def fill(self, t0=0, t1=1 << 62, skip=()) -> "State":
        """Source stores with the synthetic payload, tensors [t0, t1); devices in `skip` (a
        recovery's failed devices) stay empty."""
        out = C.c_void_p()
        w = np.array([d[0] for d in skip] + [0], np.uint32)
        l = np.array([d[1] for d in skip] + [0], np.uint32)
        self.o._chk(self.o.lib.orc_state_fill(C.c_void_p(self.h), C.c_int64(t0), C.c_int64(t1), C.c_int(len(skip)),
                                              w.ctypes.data_as(C.c_void_p), l.ctypes.data_as(C.c_void_p),
                                              C.byref(out)))
        return State(self.o, out.value, self)

    def digest(self, state: "State", t: int) -> int:
        d = C.c_uint64()
        self.o._chk(self.o.lib.orc_state_digest(C.c_void_p(self.h), C.c_void_p(state.h), C.c_int(t), C.byref(d)))
        return d.value


class Plan(_Handle):
    _free = "orc_plan_free"

    def __init__(self, o, h, a, b):
        super().__init__(o, h)
        self.a, self.b = a, b

    def text(self) -> str:
        n = self.o.lib.orc_plan_text(C.c_void_p(self.h), None, 0)
        buf = C.create_string_buffer(int(n))
        self.o.lib.orc_plan_text(C.c_void_p(self.h), buf, n)
        return buf.value.decode()

    def stats(self) -> dict:
        s = np.zeros(8, np.uint64)
        self.o._chk(self.o.lib.orc_plan_stats(C.c_void_p(self.h), s.ctypes.data_as(C.c_void_p)))
        keys = ["n_split", "n_move", "n_merge", "moved_bytes", "relayout_bytes", "kept_bytes", "dst_bytes"]
        return {k: int(v) for k, v in zip(keys, s)}

    def cost(self) -> dict:
        cap = 4096
        w = np.zeros(cap, np.uint32)
        l = np.zeros(cap, np.uint32)
        i = np.zeros(cap, np.uint64)
        e = np.zeros(cap, np.uint64)
        n = C.c_int()
        self.o._chk(self.o.lib.orc_plan_cost(C.c_void_p(self.h), C.c_int(cap), w.ctypes.data_as(C.c_void_p),
                                             l.ctypes.data_as(C.c_void_p), i.ctypes.data_as(C.c_void_p),
                                             e.ctypes.data_as(C.c_void_p), C.byref(n)))
        return {(int(w[k]), int(l[k])): (int(i[k]), int(e[k])) for k in range(n.value)}

    def apply(self, src: "State", n_threads=1, t0=0, t1=1 << 62, per_device=False):
        """apply_plan distributed; per_device: one task per destination device
        (SPEC.md:504), else every thread drains a shared (destination, tensor, cell) queue."""
        out = C.c_void_p()
        secs = C.c_double()
        moved = C.c_uint64()
        local = C.c_uint64()
        self.o._chk(self.o.lib.orc_apply(C.c_void_p(self.h), C.c_void_p(src.h), C.c_int64(t0), C.c_int64(t1),
                                         C.c_int(n_threads), C.c_int(1 if per_device else 0), C.byref(secs),
                                         C.byref(moved), C.byref(local), C.byref(out)))
        st = State(self.o, out.value, self.b)
        return st, dict(seconds=secs.value, moved=moved.value, local=local.value)


class State(_Handle):
    _free = "orc_state_free"

    def __init__(self, o, h, ptc):
        super().__init__(o, h)
        self.ptc = ptc

    def cell(self, dev, t, box) -> np.ndarray:
        lo, hi = _box_arrays([box])
        nb = C.c_uint64()
        self.o._chk(self.o.lib.orc_state_cell(C.c_void_p(self.h), C.c_uint32(dev[0]), C.c_uint32(dev[1]), C.c_int(t),
                                              C.c_int(len(box)), lo.ctypes.data_as(C.c_void_p),
                                              hi.ctypes.data_as(C.c_void_p), None, C.c_uint64(0), C.byref(nb)))
        out = np.zeros(max(nb.value, 1), np.uint8)
        self.o._chk(self.o.lib.orc_state_cell(C.c_void_p(self.h), C.c_uint32(dev[0]), C.c_uint32(dev[1]), C.c_int(t),
                                              C.c_int(len(box)), lo.ctypes.data_as(C.c_void_p),
                                              hi.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p),
                                              C.c_uint64(nb.value), C.byref(nb)))
        return out[: nb.value]


def _grid_args(shape, points):
    sh = np.array(list(shape) + [0], np.uint64)
    npts = np.array([len(p) for p in points] + [0], np.int32)
    pts = np.array([x for p in points for x in p] + [0], np.uint64)
    return sh, npts, pts


def _vp(a):
    return a.ctypes.data_as(C.c_void_p)


def _oracle_grid_cell(self, shape, points, index):
    sh, npts, pts = _grid_args(shape, points)
    lo, hi = np.zeros(MAXR, np.uint64), np.zeros(MAXR, np.uint64)
    self._chk(self.lib.orc_grid_cell(C.c_int(len(shape)), _vp(sh), _vp(npts), _vp(pts), C.c_uint64(index), _vp(lo), _vp(hi)))
    return [(int(lo[d]), int(hi[d])) for d in range(len(shape))]


def _oracle_grid_cell_index_of(self, shape, points, box):
    sh, npts, pts = _grid_args(shape, points)
    lo, hi = _box_arrays([box])
    out = C.c_uint64()
    self._chk(self.lib.orc_grid_cell_index_of(C.c_int(len(shape)), _vp(sh), _vp(npts), _vp(pts), C.c_int(len(box)),
                                              _vp(lo), _vp(hi), C.byref(out)))
    return out.value


def _oracle_offset_by(self, box, outer):
    lo, hi = _box_arrays([box])
    olo, ohi = _box_arrays([outer])
    rl, rh = np.zeros(MAXR, np.uint64), np.zeros(MAXR, np.uint64)
    self._chk(self.lib.orc_offset_by(C.c_int(len(box)), _vp(lo), _vp(hi), C.c_int(len(outer)), _vp(olo), _vp(ohi),
                                     _vp(rl), _vp(rh)))
    return [(int(rl[d]), int(rh[d])) for d in range(len(box))]


def _oracle_spec_resolve(self, spec, shape):
    M = (1 << 64) - 1
    box = [(M, M) if s is None else s for s in spec]
    lo, hi = _box_arrays([box])
    sh = np.array(list(shape) + [0], np.uint64)
    rl, rh = np.zeros(MAXR, np.uint64), np.zeros(MAXR, np.uint64)
    self._chk(self.lib.orc_spec_resolve(C.c_int(len(spec)), _vp(lo), _vp(hi), C.c_int(len(shape)), _vp(sh), _vp(rl), _vp(rh)))
    return [(int(rl[d]), int(rh[d])) for d in range(len(spec))]


Oracle.grid_cell = _oracle_grid_cell
Oracle.grid_cell_index_of = _oracle_grid_cell_index_of
Oracle.offset_by = _oracle_offset_by
Oracle.spec_resolve = _oracle_spec_resolve
