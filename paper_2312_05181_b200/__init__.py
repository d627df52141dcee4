"""B200-native PTC state transformation (Tenplex, arxiv 2312.05181) — Python front-end.

Thin wrappers over the C-ABI in ``include/reshard_b200.h``; every operation runs in
``libreshard_b200.so`` (host C++ planner + sm_100a CUDA kernels).  Names follow the
reference's C++ API (``reshard::slice``, ``merge``, ``SplitGrid``, ``grid_refine``) and the
SPEC modules (``build_strategy``, ``hosted_subtensors``, ``validate``, ``generate_plan``,
``recover``, ``plan_cost``, ``apply_plan``).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Iterable, Sequence

from . import _capi
from ._capi import MAXR, rs_cell_binding, rs_device, rs_range, rs_tensor

class _LazyLib:
    """Loads libreshard_b200.so on first use (so `python -m paper_2312_05181_b200.build` can
    run before it exists).  A missing or stale library raises ImportError at that point —
    there is no fallback."""

    def __getattr__(self, name):
        global lib
        real = _capi.load()
        lib = real
        return getattr(real, name)


lib = _LazyLib()


def load() -> None:
    """Force-load the native library now (raises ImportError when it is missing)."""
    getattr(lib, "rs_build_info")

F32, F16, I64, U8, BF16 = 0, 1, 2, 3, 4
WIDTH = {F32: 4, F16: 2, I64: 8, U8: 1, BF16: 2}
FP32_ADAM, MIXED_ADAM, FP32_PARAM = 0, 1, 2
LAYER_PRE, LAYER_POST = -1, -2
HOST_SKIP_UNREAD = 1  # RS_HOST_SKIP_UNREAD (run_host flags)


class ReshardError(Exception):
    """Error carrying the reference's Errc (error.hpp:8-48) plus the appended codes."""

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code
        self.name = _capi.ERRC[code] if 0 <= code < len(_capi.ERRC) else "Unknown"


def _chk(rc: int) -> None:
    if rc != 0:
        raise ReshardError(rc - 1, lib.rs_last_error().decode())


def _u64(vals) -> C.Array:
    vals = list(vals)
    return (C.c_uint64 * max(len(vals), 1))(*vals)


def _i32(vals) -> C.Array:
    vals = list(vals)
    return (C.c_int32 * max(len(vals), 1))(*vals)


def _range(box) -> rs_range:
    r = rs_range()
    box = list(box)
    r.rank = len(box)
    for i, (a, z) in enumerate(box[:MAXR]):
        r.lo[i], r.hi[i] = int(a), int(z)
    return r


def _box(r: rs_range):
    return [(int(r.lo[i]), int(r.hi[i])) for i in range(r.rank)]


def _devs(devs) -> C.Array:
    devs = list(devs)
    arr = (rs_device * max(len(devs), 1))()
    for i, (w, l) in enumerate(devs):
        arr[i].worker, arr[i].local = int(w), int(l)
    return arr


def fnv1a64(data: bytes) -> int:
    return int(lib.rs_fnv1a64(data, len(data)))


def payload_seed(path: str) -> int:
    return int(lib.rs_payload_seed(path.encode()))


def build_info() -> str:
    return lib.rs_build_info().decode()


# ---- box algebra -------------------------------------------------------------------------
def range_parse(text: str):
    r = rs_range()
    _chk(lib.rs_range_parse(text.encode(), C.byref(r)))
    return _box(r)


def range_format(box) -> str:
    buf = C.create_string_buffer(1024)
    _chk(lib.rs_range_format(C.byref(_range(box)), buf, 1024))
    return buf.value.decode()


def grid_cells(shape, points):
    cap = 1
    for p in points:
        cap *= len(p) + 1
    cells = (rs_range * max(cap, 1))()
    n = C.c_int()
    _chk(lib.rs_grid_cells(len(shape), _u64(shape), _i32(len(p) for p in points), _u64(x for p in points for x in p),
                           cap, cells, C.byref(n)))
    return [_box(cells[i]) for i in range(min(n.value, cap))]


def _grid_out(rank, npts, pts):
    res, k = [], 0
    for d in range(rank):
        res.append([int(pts[k + i]) for i in range(npts[d])])
        k += npts[d]
    return res


def grid_refine(a, b):
    tot = sum(len(p) for p in a) + sum(len(p) for p in b)
    npts, pts = _i32([0] * max(len(a), 1)), _u64([0] * max(tot, 1))
    _chk(lib.rs_grid_refine(len(a), _i32(len(p) for p in a), _u64(x for p in a for x in p), len(b),
                            _i32(len(p) for p in b), _u64(x for p in b for x in p), npts, pts))
    return _grid_out(len(a), npts, pts)


def even_split(shape, dim, ways):
    npts, pts = _i32([0] * max(len(shape), 1)), _u64([0] * max(int(ways), 1))
    _chk(lib.rs_even_split(len(shape), _u64(shape), int(dim), int(ways), npts, pts))
    return _grid_out(len(shape), npts, pts)


def grid_cell(shape, points, index):
    """SplitGrid::cell (split_grid.cpp:88-101): the index-th cell, last dim fastest."""
    r = rs_range()
    _chk(lib.rs_grid_cell(len(shape), _u64(shape), _i32(len(p) for p in points), _u64(x for p in points for x in p),
                          int(index), C.byref(r)))
    return _box(r)


def grid_cell_index_of(shape, points, box):
    """SplitGrid::cell_index_of (split_grid.cpp:103-117): index of the cell holding `box`."""
    idx = C.c_uint64()
    _chk(lib.rs_grid_cell_index_of(len(shape), _u64(shape), _i32(len(p) for p in points),
                                   _u64(x for p in points for x in p), C.byref(_range(box)), C.byref(idx)))
    return idx.value


def range_offset_by(box, outer):
    """Range::offset_by (range.cpp:80-90): box given relative to `outer`, made absolute."""
    r = rs_range()
    _chk(lib.rs_range_offset_by(C.byref(_range(box)), C.byref(_range(outer)), C.byref(r)))
    return _box(r)


def range_valid_for(box, shape) -> bool:
    ok = C.c_int32()
    _chk(lib.rs_range_valid_for(C.byref(_range(box)), len(shape), _u64(shape), C.byref(ok)))
    return bool(ok.value)


def rangespec_resolve(spec: str, shape):
    """RangeSpec::parse(spec).resolve(shape) (range.cpp:153-193): ':' binds the full extent."""
    r = rs_range()
    _chk(lib.rs_rangespec_resolve(spec.encode(), len(shape), _u64(shape), C.byref(r)))
    return _box(r)


def dtype_from_name(name: str) -> int:
    code = C.c_int32()
    _chk(lib.rs_dtype_from_name(name.encode(), C.byref(code)))
    return code.value


# ---- device runtime ------------------------------------------------------------------------
def device_count() -> int:
    n = C.c_int()
    _chk(lib.rs_device_count(C.byref(n)))
    return n.value


class Context:
    """The GPUs this process drives, out of a world of `world` GPUs."""

    def __init__(self, world: int = 1, world_ids: Sequence[int] = (0,), cuda_devices: Sequence[int] | None = None):
        cuda_devices = list(world_ids) if cuda_devices is None else list(cuda_devices)
        h = C.c_void_p()
        _chk(lib.rs_init(world, len(world_ids), _i32(world_ids), _i32(cuda_devices), C.byref(h)))
        self.h, self.world, self.world_ids = h.value, world, list(world_ids)

    def __del__(self):
        if getattr(self, "h", None):
            lib.rs_destroy(self.h)
            self.h = None

    def malloc(self, gpu: int, nbytes: int) -> int:
        p = C.c_void_p()
        _chk(lib.rs_malloc(self.h, gpu, nbytes, C.byref(p)))
        return p.value

    def free(self, gpu: int, ptr: int) -> None:
        _chk(lib.rs_free(self.h, gpu, ptr))

    def htod(self, gpu: int, dst: int, src, nbytes: int) -> None:
        _chk(lib.rs_memcpy_htod(self.h, gpu, dst, src, nbytes))

    def dtoh(self, gpu: int, dst, src: int, nbytes: int) -> None:
        _chk(lib.rs_memcpy_dtoh(self.h, gpu, dst, src, nbytes))

    def memset(self, gpu: int, dst: int, value: int, nbytes: int) -> None:
        _chk(lib.rs_memset(self.h, gpu, dst, value, nbytes))

    def sync(self, gpu: int) -> None:
        _chk(lib.rs_sync(self.h, gpu))

    def ipc_handle(self, gpu: int, ptr: int) -> bytes:
        buf = C.create_string_buffer(64)
        _chk(lib.rs_ipc_get_handle(self.h, gpu, ptr, buf))
        return buf.raw

    def ipc_open(self, gpu: int, handle: bytes) -> int:
        p = C.c_void_p()
        _chk(lib.rs_ipc_open_handle(self.h, gpu, C.create_string_buffer(handle, 64), C.byref(p)))
        return p.value


class Event:
    """A stream event on one GPU of a context: an interprocess event (create: new + its 64-byte
    handle in .handle; open: a peer rank's handle) or a timing event; record / wait enqueue on
    the GPU's context stream (rs_event_*)."""

    def __init__(self, ctx: Context, gpu: int, kind: str = "timing", handle: bytes | None = None):
        h = C.c_void_p()
        self.ctx, self.gpu, self.handle = ctx, gpu, None
        if kind == "ipc" and handle is None:
            buf = C.create_string_buffer(64)
            _chk(lib.rs_ipc_event_create(ctx.h, gpu, buf, C.byref(h)))
            self.handle = buf.raw
        elif kind == "ipc":
            _chk(lib.rs_ipc_event_open(ctx.h, gpu, C.create_string_buffer(handle, 64), C.byref(h)))
        else:
            _chk(lib.rs_timing_event_create(ctx.h, gpu, C.byref(h)))
        self.h = h.value

    def __del__(self):
        if getattr(self, "h", None):
            lib.rs_event_destroy(self.h)
            self.h = None

    def record(self) -> None:
        _chk(lib.rs_event_record(self.ctx.h, self.gpu, self.h))

    def wait(self) -> None:
        _chk(lib.rs_event_wait(self.ctx.h, self.gpu, self.h))

    def elapsed_since(self, start: "Event") -> float:
        ms = C.c_float()
        _chk(lib.rs_event_elapsed(start.h, self.h, C.byref(ms)))
        return ms.value


def host_alloc(nbytes: int) -> int:
    p = C.c_void_p()
    _chk(lib.rs_host_alloc(nbytes, C.byref(p)))
    return p.value


def host_free(ptr: int) -> None:
    _chk(lib.rs_host_free(ptr))


@dataclass
class DeviceTensor:
    """A dense row-major tensor in device memory (caller-owned)."""
    dtype: int
    shape: tuple
    ptr: int

    def c(self) -> rs_tensor:
        t = rs_tensor()
        t.dtype, t.rank, t.data = self.dtype, len(self.shape), self.ptr
        for i, e in enumerate(self.shape[:MAXR]):
            t.shape[i] = int(e)
        return t


def slice(ctx: Context, gpu: int, t: DeviceTensor, box, out: int) -> None:
    """reshard::slice (tensor.cpp:61-78) on device: out <- t[box] (dense)."""
    _chk(lib.rs_slice(ctx.h, gpu, C.byref(t.c()), C.byref(_range(box)), out))


def merge(ctx: Context, gpu: int, parts: Sequence[tuple], target_shape, out: int) -> None:
    """reshard::merge (tensor.cpp:80-114) on device: parts = [(box, DeviceTensor), ...]."""
    n = len(parts)
    rngs = (rs_range * max(n, 1))(*[_range(b) for b, _ in parts])
    ts = (rs_tensor * max(n, 1))(*[t.c() for _, t in parts])
    _chk(lib.rs_merge(ctx.h, gpu, n, rngs, ts, len(target_shape), _u64(target_shape), out))


def broadcast(ctx: Context, gpu: int, src_ptr: int, dst_ptrs: Sequence[int], nbytes: int) -> dict:
    """DP replication as one push (rs_broadcast): src -> every dst pointer, source read once
    per 4 destinations (TMA fan-out tiles when aligned)."""
    n = len(dst_ptrs)
    arr = (C.c_void_p * max(n, 1))(*dst_ptrs)
    t = _capi.rs_timing()
    _chk(lib.rs_broadcast(ctx.h, gpu, src_ptr, n, arr, nbytes, C.byref(t)))
    return dict(ms=t.ms, tiles=t.tiles, bytes=t.bytes, read_bytes=t.read_bytes, launches=t.launches)


def slice_host(ctx: Context, gpu: int, dtype: int, shape, payload: bytes, box) -> bytes:
    """The reference's value-level slice (tensor.hpp:40-42) on host bytes, through the GPU."""
    import numpy as np

    src = np.frombuffer(payload, np.uint8).copy() if len(payload) else np.zeros(1, np.uint8)
    w = WIDTH.get(dtype, 1)
    n = int(np.prod([b - a for a, b in box])) * w if box else w
    out = np.zeros(max(n, 1), np.uint8)
    t = DeviceTensor(dtype, tuple(shape), src.ctypes.data)
    _chk(lib.rs_slice_host(ctx.h, gpu, C.byref(t.c()), C.byref(_range(box)), out.ctypes.data))
    return out[:n].tobytes()


def merge_host(ctx: Context, gpu: int, parts: Sequence[tuple], target_shape, dtype_hint: int = 0) -> bytes:
    """The reference's value-level merge (tensor.hpp:44-47) on host bytes:
    parts = [(box, dtype, shape, payload bytes), ...]."""
    import numpy as np

    keep = [np.frombuffer(p, np.uint8).copy() if len(p) else np.zeros(1, np.uint8) for _, _, _, p in parts]
    n = len(parts)
    rngs = (rs_range * max(n, 1))(*[_range(b) for b, _, _, _ in parts])
    ts = (rs_tensor * max(n, 1))(*[DeviceTensor(dt, tuple(sh), k.ctypes.data).c() for (_, dt, sh, _), k in zip(parts, keep)])
    dt = parts[0][1] if parts else dtype_hint
    w = WIDTH.get(dt, 1)
    nbytes = int(np.prod(target_shape)) * w if len(target_shape) else w
    out = np.zeros(max(nbytes, 1), np.uint8)
    _chk(lib.rs_merge_host(ctx.h, gpu, n, rngs, ts, len(target_shape), _u64(target_shape), out.ctypes.data))
    return out[:nbytes].tobytes()


# ---- collection description ------------------------------------------------------------------
class Catalog:
    def __init__(self, handle=None):
        if handle is None:
            h = C.c_void_p()
            _chk(lib.rs_catalog_create(C.byref(h)))
            handle = h.value
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None):
            lib.rs_catalog_destroy(self.h)
            self.h = None

    @classmethod
    def gpt(cls, hidden, layers, seq, vocab, kind=FP32_ADAM) -> "Catalog":
        h = C.c_void_p()
        _chk(lib.rs_catalog_gpt(hidden, layers, seq, vocab, kind, C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_entries(cls, entries: Iterable[tuple]) -> "Catalog":
        c = cls()
        for e in entries:
            c.add(*e)
        return c

    def add(self, path: str, dtype: int, shape, tp_dim: int = -1, layer: int = 0) -> None:
        _chk(lib.rs_catalog_add(self.h, path.encode(), dtype, len(shape), _u64(shape), tp_dim, layer))

    def __len__(self) -> int:
        return lib.rs_catalog_size(self.h)

    def entry(self, i: int):
        name = C.create_string_buffer(512)
        dt, rk, tp, ly = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        sh = (C.c_uint64 * MAXR)()
        _chk(lib.rs_catalog_get(self.h, i, name, 512, C.byref(dt), C.byref(rk), sh, C.byref(tp), C.byref(ly)))
        return (name.value.decode(), dt.value, tuple(int(sh[d]) for d in range(rk.value)), tp.value, ly.value)

    def entries(self):
        return [self.entry(i) for i in range(len(self))]

    def nbytes(self) -> int:
        return int(lib.rs_catalog_bytes(self.h))

    def build_strategy(self, devices, tp=1, pp=1, dp=1) -> "PTC":
        devices = [tuple(d) for d in devices]
        h = C.c_void_p()
        _chk(lib.rs_build_strategy(self.h, len(devices), _devs(devices), tp, pp, dp, C.byref(h)))
        return PTC(h.value, self, devices, (tp, pp, dp))


def build_strategy(catalog: Catalog, devices, tp=1, pp=1, dp=1) -> "PTC":
    """device (dp, pp, tp) = devices[dp*P*T + pp*T + tp]."""
    return catalog.build_strategy(devices, tp, pp, dp)


class PTC:
    def __init__(self, h, catalog, devices, degrees):
        self.h, self.catalog, self.devices, self.degrees = h, catalog, devices, degrees

    def __del__(self):
        if getattr(self, "h", None):
            lib.rs_ptc_destroy(self.h)
            self.h = None

    def validate(self):
        buf = C.create_string_buffer(1 << 16)
        n = C.c_int()
        _chk(lib.rs_validate(self.h, buf, 1 << 16, C.byref(n)))
        return [x for x in buf.value.decode().split("\n") if x]

    def hosted_subtensors(self, dev):
        cap = 1 << 16
        ts = (C.c_int32 * cap)()
        cells = (rs_range * cap)()
        n = C.c_int()
        d = rs_device(int(dev[0]), int(dev[1]))
        _chk(lib.rs_hosted_subtensors(self.h, d, cap, ts, cells, C.byref(n)))
        return [(int(ts[i]), _box(cells[i])) for i in range(min(n.value, cap))]

    def cell(self, tensor: int, index: int):
        r = rs_range()
        _chk(lib.rs_ptc_cell(self.h, tensor, index, C.byref(r)))
        return _box(r)

    def cell_count(self, tensor: int) -> int:
        n = C.c_int()
        _chk(lib.rs_ptc_cell_count(self.h, tensor, C.byref(n)))
        return n.value

    def set_alpha(self, partition, devices):
        devices = list(devices)
        _chk(lib.rs_ptc_set_alpha(self.h, partition, len(devices), _devs(devices)))

    def set_sigma(self, tensor, points):
        _chk(lib.rs_ptc_set_sigma(self.h, tensor, len(points), _i32(len(p) for p in points),
                                  _u64(x for p in points for x in p)))


def hosted_subtensors(ptc: PTC, dev):
    return ptc.hosted_subtensors(dev)


def validate(ptc: PTC):
    return ptc.validate()


# ---- planner --------------------------------------------------------------------------------
class Plan:
    def __init__(self, h, src: PTC, dst: PTC):
        self.h, self.src, self.dst = h, src, dst

    def __del__(self):
        if getattr(self, "h", None):
            lib.rs_plan_destroy(self.h)
            self.h = None

    def stats(self) -> dict:
        s = _capi.rs_plan_stats()
        _chk(lib.rs_plan_get_stats(self.h, C.byref(s)))
        return {k: int(getattr(s, k)) for k, _ in s._fields_}

    def cost(self) -> dict:
        cap = 4096
        devs = (rs_device * cap)()
        ing, eg = (C.c_uint64 * cap)(), (C.c_uint64 * cap)()
        n = C.c_int()
        _chk(lib.rs_plan_cost(self.h, cap, devs, ing, eg, C.byref(n)))
        return {(int(devs[i].worker), int(devs[i].local)): (int(ing[i]), int(eg[i])) for i in range(n.value)}

    def cost_central(self, central) -> dict:
        cap = 4096
        devs = (rs_device * cap)()
        ing, eg = (C.c_uint64 * cap)(), (C.c_uint64 * cap)()
        n = C.c_int()
        _chk(lib.rs_plan_cost_central(self.h, rs_device(*central), cap, devs, ing, eg, C.byref(n)))
        return {(int(devs[i].worker), int(devs[i].local)): (int(ing[i]), int(eg[i])) for i in range(n.value)}

    def text(self) -> str:
        n = lib.rs_plan_text(self.h, None, 0)
        buf = C.create_string_buffer(int(n))
        lib.rs_plan_text(self.h, buf, n)
        return buf.value.decode()


def generate_plan(src: PTC, dst: PTC) -> Plan:
    h = C.c_void_p()
    _chk(lib.rs_generate_plan(src.h, dst.h, C.byref(h)))
    return Plan(h.value, src, dst)


def recover(src: PTC, failed, dst: PTC) -> Plan:
    failed = list(failed)
    h = C.c_void_p()
    _chk(lib.rs_recover(src.h, len(failed), _devs(failed), dst.h, C.byref(h)))
    return Plan(h.value, src, dst)


def plan_cost(plan: Plan) -> dict:
    return plan.cost()


def choose_source(candidates, egress, dst):
    out = rs_device()
    _chk(lib.rs_choose_source(len(candidates), _devs(candidates), _u64(egress), rs_device(*dst), C.byref(out)))
    return (int(out.worker), int(out.local))


# ---- executor (apply_plan) ---------------------------------------------------------------------
@dataclass
class Binding:
    gpu: int
    arena: int  # 0 src, 1 dst
    offset: int
    nbytes: int


class Executor:
    """apply_plan data plane: arenas per GPU, one tile-copy kernel per source GPU."""

    def __init__(self, ctx: Context, plan: Plan, src_gpu: Sequence[int], dst_gpu: Sequence[int],
                 tile_bytes: int = 256 << 10, window: tuple[int, int] | None = None, central: int | None = None):
        """central=g: apply_plan's central mode, every moved fragment staged
        on GPU g; otherwise distributed mode (push from each source GPU)."""
        h = C.c_void_p()
        if central is not None:
            if window is not None:
                raise ValueError("central mode runs the whole catalog (no window)")
            _chk(lib.rs_executor_create_central(ctx.h, plan.h, _i32(src_gpu), _i32(dst_gpu), tile_bytes, int(central),
                                                C.byref(h)))
        elif window is None:
            _chk(lib.rs_executor_create(ctx.h, plan.h, _i32(src_gpu), _i32(dst_gpu), tile_bytes, C.byref(h)))
        else:
            _chk(lib.rs_executor_create_window(ctx.h, plan.h, _i32(src_gpu), _i32(dst_gpu), tile_bytes,
                                               int(window[0]), int(window[1]), C.byref(h)))
        self.h, self.ctx, self.plan = h.value, ctx, plan
        self.arenas: dict[int, tuple[int, int]] = {}
        self._owned: list[tuple[int, int]] = []

    def __del__(self):
        if getattr(self, "h", None):
            lib.rs_executor_destroy(self.h)
            self.h = None
        for gpu, p in getattr(self, "_owned", []):
            try:
                self.ctx.free(gpu, p)
            except Exception:
                pass
        self._owned = []

    def arena_bytes(self, gpu: int) -> tuple[int, int]:
        s, d = C.c_uint64(), C.c_uint64()
        _chk(lib.rs_executor_arena_bytes(self.h, gpu, C.byref(s), C.byref(d)))
        return s.value, d.value

    def staging_bytes(self) -> int:
        b = C.c_uint64()
        _chk(lib.rs_executor_staging_bytes(self.h, C.byref(b)))
        return b.value

    def bind(self, gpu: int, src_ptr: int, dst_ptr: int) -> None:
        _chk(lib.rs_executor_bind(self.h, gpu, src_ptr, dst_ptr))
        self.arenas[gpu] = (src_ptr, dst_ptr)

    def allocate_local(self) -> None:
        """Allocate and bind both arenas of every GPU this context drives."""
        for g in self.ctx.world_ids:
            s, d = self.arena_bytes(g)
            sp, dp = self.ctx.malloc(g, max(s, 256)), self.ctx.malloc(g, max(d, 256))
            self._owned += [(g, sp), (g, dp)]
            self.bind(g, sp, dp)

    def prepare(self) -> None:
        _chk(lib.rs_executor_prepare(self.h))

    def run(self) -> None:
        _chk(lib.rs_executor_run(self.h))

    def wait(self) -> list[dict]:
        cap = 64
        t = (_capi.rs_timing * cap)()
        n = C.c_int()
        _chk(lib.rs_executor_wait(self.h, cap, t, C.byref(n)))
        return [dict(ms=t[i].ms, tiles=t[i].tiles, bytes=t[i].bytes, launches=t[i].launches, read_bytes=t[i].read_bytes)
                for i in range(n.value)]

    def apply(self) -> list[dict]:
        self.run()
        return self.wait()

    def run_host(self, gpu: int, host_src: int, host_dst: int, skip_unread: bool = False) -> dict:
        """skip_unread: upload only the source ranges the tiles read (RS_HOST_SKIP_UNREAD)."""
        t = _capi.rs_timing()
        if skip_unread:
            _chk(lib.rs_executor_run_host_flags(self.h, gpu, host_src, host_dst, HOST_SKIP_UNREAD, C.byref(t)))
        else:
            _chk(lib.rs_executor_run_host(self.h, gpu, host_src, host_dst, C.byref(t)))
        return dict(ms=t.ms, tiles=t.tiles, bytes=t.bytes, launches=t.launches, read_bytes=t.read_bytes)

    def host_upload_bytes(self, gpu: int, skip_unread: bool = False) -> int:
        b = C.c_uint64()
        _chk(lib.rs_executor_host_upload_bytes(self.h, gpu, HOST_SKIP_UNREAD if skip_unread else 0, C.byref(b)))
        return b.value

    def host_phase(self, gpu: int, phase: int, host_buf: int = 0) -> None:
        _chk(lib.rs_executor_host_phase(self.h, gpu, phase, host_buf))

    def host_elapsed(self, gpu: int) -> float:
        ms = C.c_float()
        _chk(lib.rs_executor_host_elapsed(self.h, gpu, C.byref(ms)))
        return ms.value

    def world_ms(self) -> float:
        """The last wait()'s world time: common start -> last local GPU done (peer pushes included)."""
        ms = C.c_float()
        _chk(lib.rs_executor_world_ms(self.h, C.byref(ms)))
        return ms.value

    def run_host_world(self, host_src: Sequence[int], host_dst: Sequence[int]) -> float:
        """End to end over every local GPU: H2D of all src arenas | kernels | D2H of all dst
        arenas, from one common start (ms).  One pinned host buffer pair per world GPU."""
        n = self.ctx.world
        hs, hd = (C.c_void_p * n)(*[p or None for p in host_src]), (C.c_void_p * n)(*[p or None for p in host_dst])
        ms = C.c_float()
        _chk(lib.rs_executor_run_host_world(self.h, n, hs, hd, C.byref(ms)))
        return ms.value

    def digests(self, side: int = 1, replica: int = 0) -> dict:
        """{tensor: FNV-1a-64 of the reassembled base tensor} over side 0 (source cells) or 1
        (destination cells), from DP copy `replica` of each cell (0 first, -1 last) — the
        ExecutionReport verification digest; tensors with a cell on no local
        GPU are left out."""
        n = C.c_int()
        _chk(lib.rs_executor_digests(self.h, side, replica, 0, None, None, None, C.byref(n)))
        m = max(n.value, 1)
        tt, ff, ok = (C.c_int32 * m)(), (C.c_uint64 * m)(), (C.c_int32 * m)()
        _chk(lib.rs_executor_digests(self.h, side, replica, n.value, tt, ff, ok, C.byref(n)))
        return {int(tt[i]): int(ff[i]) for i in range(n.value) if ok[i]}

    def fill_sources(self) -> None:
        _chk(lib.rs_executor_fill_sources(self.h))

    def verify(self) -> int:
        bad = C.c_uint64()
        _chk(lib.rs_executor_verify(self.h, C.byref(bad)))
        return bad.value

    def src_cells(self) -> list[Binding]:
        n = C.c_int()
        _chk(lib.rs_executor_src_cells(self.h, 0, None, C.byref(n)))
        arr = (rs_cell_binding * max(n.value, 1))()
        _chk(lib.rs_executor_src_cells(self.h, n.value, arr, C.byref(n)))
        return [Binding(arr[i].gpu, arr[i].arena, arr[i].offset, arr[i].bytes) for i in range(n.value)]

    def dst_cells(self) -> list[tuple[int, int, int, Binding]]:
        """[(to-device ordinal, tensor, cell index, binding)] in plan order."""
        n = C.c_int()
        _chk(lib.rs_executor_dst_cells(self.h, 0, None, None, None, None, C.byref(n)))
        m = max(n.value, 1)
        arr = (rs_cell_binding * m)()
        dv, tt, cc = (C.c_int32 * m)(), (C.c_int32 * m)(), (C.c_int32 * m)()
        _chk(lib.rs_executor_dst_cells(self.h, n.value, arr, dv, tt, cc, C.byref(n)))
        return [(dv[i], tt[i], cc[i], Binding(arr[i].gpu, arr[i].arena, arr[i].offset, arr[i].bytes))
                for i in range(n.value)]

    def read_bytes(self, gpu: int) -> int:
        b = C.c_uint64()
        _chk(lib.rs_executor_read_bytes(self.h, gpu, C.byref(b)))
        return b.value

    def bytes_to(self, gpu: int) -> list[int]:
        """Bytes GPU `gpu`'s tiles write into each world GPU (its egress row; own entry = local)."""
        n = self.ctx.world
        arr = (C.c_uint64 * n)()
        _chk(lib.rs_executor_bytes_to(self.h, gpu, n, arr))
        return list(arr)

    def tiles(self, gpu: int) -> tuple[int, int]:
        t, b = C.c_uint64(), C.c_uint64()
        _chk(lib.rs_executor_tiles(self.h, gpu, C.byref(t), C.byref(b)))
        return t.value, b.value

    def cell_ptr(self, b: Binding) -> int:
        return self.arenas[b.gpu][b.arena] + b.offset


def apply_plan(ctx: Context, plan: Plan, src_gpu=None, dst_gpu=None) -> Executor:
    """Convenience: all logical devices on the context's GPUs round-robin, arenas allocated,
    sources filled with the synthetic payload, plan executed once."""
    src_gpu = src_gpu if src_gpu is not None else [0] * len(plan.src.devices)
    dst_gpu = dst_gpu if dst_gpu is not None else [0] * len(plan.dst.devices)
    ex = Executor(ctx, plan, src_gpu, dst_gpu)
    ex.allocate_local()
    ex.prepare()
    ex.fill_sources()
    ex.apply()
    return ex


# ---- dataset index repartitioning -------------------------------------------
def shuffle_epoch(n: int, seed: int, epoch: int):
    import numpy as np

    perm = np.empty(max(n, 1), np.uint64)
    _chk(lib.rs_shuffle_epoch(n, seed, epoch, perm.ctypes.data))
    return perm[:n]


def repartition_count(n, global_batch, at_step, new_dp, rank) -> int:
    c = C.c_uint64()
    _chk(lib.rs_repartition_count(n, global_batch, at_step, new_dp, rank, C.byref(c)))
    return c.value


def repartition_position(n, global_batch, at_step, new_dp, rank, k) -> int:
    c = C.c_uint64()
    _chk(lib.rs_repartition_position(n, global_batch, at_step, new_dp, rank, k, C.byref(c)))
    return c.value


def locate_sample(n, global_batch, at_step, new_dp, rank, k, perm, samples, file_class):
    """(file, offset, length, locator class) of the rank's k-th remaining sample (host arrays)."""
    import numpy as np

    out = (C.c_uint64 * 4)()
    perm = np.ascontiguousarray(perm, np.uint64)
    samples = np.ascontiguousarray(samples, np.uint64)
    file_class = np.ascontiguousarray(file_class, np.uint8)
    _chk(lib.rs_locate_sample(n, global_batch, at_step, new_dp, rank, k, perm.ctypes.data, samples.ctypes.data,
                              file_class.ctypes.data, out))
    return tuple(int(x) for x in out)


class Partition:
    """Device buffers of one rank's repartition output (K5)."""

    def __init__(self, ctx: Context, gpu: int, count: int):
        self.ctx, self.gpu, self.count = ctx, gpu, count
        n = max(count, 1)
        self.pos = ctx.malloc(gpu, 8 * n)
        self.ent = ctx.malloc(gpu, 24 * n)
        self.boff = ctx.malloc(gpu, 8 * n)
        self.queue = [ctx.malloc(gpu, 4 * n) for _ in range(3)]
        self.qcount = ctx.malloc(gpu, 24)
        sb = C.c_uint64()
        _chk(lib.rs_repartition_scratch_bytes(count, C.byref(sb)))
        self.scratch = ctx.malloc(gpu, max(sb.value, 256))

    def c(self):
        o = _capi.rs_partition_out()
        o.pos, o.ent, o.boff, o.qcount = self.pos, self.ent, self.boff, self.qcount
        for i in range(3):
            o.queue[i] = self.queue[i]
        return o

    def free(self):
        for p in [self.pos, self.ent, self.boff, self.qcount, self.scratch, *self.queue]:
            self.ctx.free(self.gpu, p)

    def fetch(self) -> dict:
        import numpy as np

        n = self.count
        out = {}
        for name, ptr, dt, width in [("pos", self.pos, np.uint64, 1), ("ent", self.ent, np.uint64, 3),
                                     ("boff", self.boff, np.uint64, 1)]:
            a = np.empty(max(n * width, 1), dt)
            self.ctx.dtoh(self.gpu, a.ctypes.data, ptr, n * width * 8)
            out[name] = a[: n * width].reshape(n, width) if width > 1 else a[:n]
        qc = np.empty(3, np.uint64)
        self.ctx.dtoh(self.gpu, qc.ctypes.data, self.qcount, 24)
        out["qcount"] = [int(x) for x in qc]
        qs = []
        for c in range(3):
            q = np.empty(max(int(qc[c]), 1), np.uint32)
            if qc[c]:
                self.ctx.dtoh(self.gpu, q.ctypes.data, self.queue[c], int(qc[c]) * 4)
            qs.append(q[: int(qc[c])])
        out["qidx"] = np.concatenate(qs) if n else np.empty(0, np.uint32)
        return out


def repartition_batch(ctx: Context, gpu: int, perm_ptr: int, samples_ptr: int, n: int, global_batch: int,
                      jobs: Sequence[tuple[int, int, int, int, "Partition"]], entry_bytes: int = 24) -> dict:
    """K5 for several ranks on one GPU: jobs = [(at_step, new_dp, rank, class_ptr, partition)]
    (rs_repartition_batch: one launch per pass for every rank; RESHARD_K5_FUSE=0 the two-stream
    schedule).  ms: whole batch; gather_ms: the gather pass(es); per_job: each rank's
    gather-pass ms when unfused (0 when fused)."""
    idx = _capi.rs_dataset_index(perm_ptr, samples_ptr, None, n, entry_bytes)
    arr = (_capi.rs_repartition_job * max(len(jobs), 1))()
    for i, (at, dp, d, cls, part) in enumerate(jobs):
        arr[i].at_step, arr[i].new_dp, arr[i].rank, arr[i].file_class = at, dp, d, cls
        arr[i].out, arr[i].scratch = part.c(), part.scratch
    per = (_capi.rs_timing * max(len(jobs), 1))()
    t = _capi.rs_timing()
    _chk(lib.rs_repartition_batch(ctx.h, gpu, C.byref(idx), global_batch, arr, len(jobs), per, C.byref(t)))
    return dict(ms=t.ms, tiles=t.tiles, bytes=t.bytes, launches=t.launches, gather_ms=t.main_ms,
                per_job=[per[i].main_ms for i in range(len(jobs))])


def repartition(ctx: Context, gpu: int, perm_ptr: int, samples_ptr: int, class_ptr: int, n: int, global_batch: int,
                at_step: int, new_dp: int, rank: int, part: "Partition", entry_bytes: int = 24) -> dict:
    """K5 for one rank.  entry_bytes 24: samples_ptr holds the packed reference records;
    32: the padded device layout from dataset_index_pad (same outputs)."""
    idx = _capi.rs_dataset_index(perm_ptr, samples_ptr, class_ptr, n, entry_bytes)
    t = _capi.rs_timing()
    out = part.c()
    _chk(lib.rs_repartition(ctx.h, gpu, C.byref(idx), global_batch, at_step, new_dp, rank, C.byref(out),
                            part.scratch, C.byref(t)))
    return dict(ms=t.ms, tiles=t.tiles, bytes=t.bytes, launches=t.launches, gather_ms=t.main_ms)


def dataset_index_upload(ctx: Context, gpu: int, host_perm: int, host_samples: int, n: int, perm_ptr: int,
                         samples_ptr: int, padded_ptr: int = 0) -> dict:
    """Host -> device upload of an index (pinned host pointers; padded_ptr: also pad it)."""
    t = _capi.rs_timing()
    _chk(lib.rs_dataset_index_upload(ctx.h, gpu, host_perm, host_samples, n, perm_ptr, samples_ptr, padded_ptr or None,
                                     C.byref(t)))
    return dict(ms=t.ms, bytes=t.bytes, launches=t.launches)


class HostPartition:
    """Pinned host buffers receiving one rank's repartition output."""

    def __init__(self, count: int):
        self.count = count
        n = max(count, 1)
        self.pos, self.ent, self.boff = host_alloc(8 * n), host_alloc(24 * n), host_alloc(8 * n)
        self.queue = [host_alloc(4 * n) for _ in range(3)]
        self.qcount = host_alloc(24)

    def c(self):
        h = _capi.rs_partition_host()
        h.pos, h.ent, h.boff, h.qcount = self.pos, self.ent, self.boff, self.qcount
        for i in range(3):
            h.queue[i] = self.queue[i]
        return h

    def arrays(self) -> dict:
        import numpy as np

        n = self.count

        def view(ptr, dt, k):
            return np.ctypeslib.as_array((C.c_uint8 * max(k * np.dtype(dt).itemsize, 1)).from_address(ptr)).view(dt)[:k]

        qc = [int(x) for x in view(self.qcount, np.uint64, 3)]
        return {"pos": view(self.pos, np.uint64, n), "ent": view(self.ent, np.uint64, 3 * n).reshape(n, 3),
                "boff": view(self.boff, np.uint64, n), "qcount": qc,
                "qidx": np.concatenate([view(self.queue[c], np.uint32, qc[c]) for c in range(3)])}

    def free(self):
        for p in [self.pos, self.ent, self.boff, self.qcount, *self.queue]:
            host_free(p)


def repartition_to_host(ctx: Context, gpu: int, perm_ptr: int, samples_ptr: int, class_ptr: int, n: int,
                        global_batch: int, at_step: int, new_dp: int, rank: int, part: "Partition",
                        host: HostPartition, entry_bytes: int = 24) -> dict:
    """K5 for one rank with its outputs read back into `host` (kernels + D2H, event-timed)."""
    idx = _capi.rs_dataset_index(perm_ptr, samples_ptr, class_ptr, n, entry_bytes)
    t = _capi.rs_timing()
    out, h = part.c(), host.c()
    _chk(lib.rs_repartition_to_host(ctx.h, gpu, C.byref(idx), global_batch, at_step, new_dp, rank, C.byref(out),
                                    part.scratch, C.byref(h), C.byref(t)))
    return dict(ms=t.ms, gather_ms=t.main_ms, d2h_bytes=t.bytes, launches=t.launches)


def dataset_index_pad(ctx: Context, gpu: int, packed_ptr: int, padded_ptr: int, n: int) -> dict:
    """Packed 24-byte index records -> padded 32-byte device layout (padded_ptr: 32 n bytes)."""
    t = _capi.rs_timing()
    _chk(lib.rs_dataset_index_pad(ctx.h, gpu, packed_ptr, padded_ptr, n, C.byref(t)))
    return dict(ms=t.ms, bytes=t.bytes, read_bytes=t.read_bytes, launches=t.launches)


def repartition_gather_probe(ctx: Context, gpu: int, perm_ptr: int, samples_ptr: int, n: int, global_batch: int,
                             at_step: int, new_dp: int, rank: int, reps: int = 3, entry_bytes: int = 24) -> dict:
    """Diagnostic: device time of K5's gathers plus its 44 output bytes per sample, coalesced and
    with no scan (the floor for any kernel producing the partition); RESHARD_PROBE=read times
    the gathers alone."""
    idx = _capi.rs_dataset_index(perm_ptr, samples_ptr, 0, n, entry_bytes)
    t = _capi.rs_timing()
    _chk(lib.rs_repartition_gather_probe(ctx.h, gpu, C.byref(idx), global_batch, at_step, new_dp, rank, reps,
                                         C.byref(t)))
    return dict(ms=t.ms, bytes=t.bytes, launches=t.launches)


def shuffle_epoch_device(ctx: Context, gpu: int, n: int, seed: int, epoch: int, perm_ptr: int) -> dict:
    """K8: the shuffle_epoch permutation computed on the GPU into perm_ptr (n x u64),
    bit-identical to the host shuffle.  Returns the timing (tiles = rounds)."""
    sb = C.c_uint64()
    _chk(lib.rs_shuffle_scratch_bytes(n, C.byref(sb)))
    scratch = ctx.malloc(gpu, max(sb.value, 256))
    try:
        t = _capi.rs_timing()
        _chk(lib.rs_shuffle_epoch_device(ctx.h, gpu, n, seed, epoch, perm_ptr, scratch, C.byref(t)))
    finally:
        ctx.free(gpu, scratch)
    return dict(ms=t.ms, rounds=t.tiles, bytes=t.bytes, launches=t.launches)
