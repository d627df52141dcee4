"""PTX1 container and per-device checkpoints over the C-ABI."""
from __future__ import annotations

import ctypes as C

from . import Executor, _chk, _u64


def _lib():
    from . import lib  # the lazily loaded libreshard_b200.so

    return lib


def ptx_encoded_size(dtype: int, shape) -> int:
    n = C.c_uint64()
    _chk(_lib().rs_ptx_encoded_size(dtype, len(shape), _u64(shape), C.byref(n)))
    return n.value


def ptx_encode(dtype: int, shape, payload: bytes) -> bytes:
    """PTX1 bytes of a host payload: magic, u8 dtype, u8 rank, u64-LE extents, payload."""
    buf = (C.c_uint8 * 80)()
    w = C.c_uint64()
    _chk(_lib().rs_ptx_encode_header(dtype, len(shape), _u64(shape), buf, 80, C.byref(w)))
    return bytes(buf[: w.value]) + bytes(payload)


def ptx_decode(data: bytes):
    """(dtype code, shape, payload) of a PTX1 buffer; ReshardError(InvalidTensor) if malformed."""
    dt, rk, hb = C.c_int32(), C.c_int32(), C.c_uint64()
    sh = (C.c_uint64 * 8)()
    raw = (C.c_uint8 * max(len(data), 1)).from_buffer_copy(data if data else b"\0")
    _chk(_lib().rs_ptx_decode_header(raw, len(data), C.byref(dt), C.byref(rk), sh, C.byref(hb)))
    return dt.value, tuple(int(sh[i]) for i in range(rk.value)), data[hb.value:]


def checkpoint_save(ex: Executor, directory: str, side: int = 0) -> dict:
    """Persist one layout of the executor (0: source cells, 1: destination cells) as
    `<dir>/<rank>/<tensor path>.ptx`."""
    f, b, s = C.c_uint64(), C.c_uint64(), C.c_double()
    _chk(_lib().rs_checkpoint_save(ex.h, side, directory.encode(), C.byref(f), C.byref(b), C.byref(s)))
    return dict(files=f.value, bytes=b.value, seconds=s.value)


def checkpoint_load(ex: Executor, directory: str) -> dict:
    """Load the executor's source layout from `<dir>/<rank>/...` (LayoutMismatch if the
    checkpoint is of another layout)."""
    f, b, s = C.c_uint64(), C.c_uint64(), C.c_double()
    _chk(_lib().rs_checkpoint_load(ex.h, directory.encode(), C.byref(f), C.byref(b), C.byref(s)))
    return dict(files=f.value, bytes=b.value, seconds=s.value)
