"""Parallelization-configuration documents over the C-ABI: the JSON
interchange format with model parallelizers, parsed into / serialized from a PTC."""
from __future__ import annotations

import ctypes as C

from . import PTC, _chk, _devs


def _lib():
    from . import lib  # the lazily loaded libreshard_b200.so

    return lib


def parse_parallel_config(doc: str, devices=None) -> PTC:
    """PTC hosting on device r exactly what rank r of `doc` declares (rank r -> devices[r],
    default (0, r)).  ReshardError: MalformedConfig / InconsistentBaseShape / CoverageGap."""
    h = C.c_void_p()
    devs = list(devices) if devices is not None else None
    _chk(_lib().rs_parse_parallel_config(doc.encode(), len(devs) if devs else 0, _devs(devs) if devs else None,
                                         C.byref(h)))
    import json

    n_ranks = len(json.loads(doc))
    devs = devs if devs is not None else [(0, r) for r in range(n_ranks)]
    return PTC(h.value, None, [tuple(d) for d in devs], None)


def serialize_parallel_config(ptc: PTC) -> str:
    lib = _lib()
    n = lib.rs_serialize_parallel_config(ptc.h, None, 0)
    if n < 0:
        _chk(1 + 12)  # MalformedConfig (path collision)
    buf = C.create_string_buffer(int(n))
    lib.rs_serialize_parallel_config(ptc.h, buf, n)
    return buf.value.decode()
