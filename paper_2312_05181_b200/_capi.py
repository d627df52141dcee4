"""ctypes declarations of include/reshard_b200.h (the C-ABI boundary).

The native library is mandatory: importing this module without ``libreshard_b200.so``
raises immediately (there is no Python or CPU fallback for any operation).
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libreshard_b200.so")
MAXR = 8

ERRC = [
    "RangeOutOfBounds", "RankMismatch", "ShapeMismatch", "TilingGap", "TilingOverlap",
    "DtypeMismatch", "InvalidSplitPoint", "InvalidTensor", "IndivisibleLayerCount",
    "IndivisibleSliceDim", "DeviceCountMismatch", "InvalidJobConfig", "MalformedConfig",
    "InconsistentBaseShape", "CoverageGap", "UnknownDevice", "CatalogMismatch",
    "UnsatisfiableFragment", "NoSource", "NotFound", "IndivisibleBatch", "StepBeyondEpoch",
    "IndexOutOfRange", "InvalidReplicaCount", "MalformedFrame", "UnknownVerb", "BadRange",
    "ConnectionFailed", "CheckpointRequired", "LayoutMismatch", "IoError", "ScriptError",
    "CudaError", "DeviceUnavailable", "InvalidArgument",
]


class rs_range(C.Structure):
    _fields_ = [("rank", C.c_int32), ("lo", C.c_uint64 * MAXR), ("hi", C.c_uint64 * MAXR)]


class rs_tensor(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("rank", C.c_int32), ("shape", C.c_uint64 * MAXR), ("data", C.c_void_p)]


class rs_device(C.Structure):
    _fields_ = [("worker", C.c_uint32), ("local", C.c_uint32)]


class rs_plan_stats(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in
                ("n_split", "n_move", "n_merge", "moved_bytes", "relayout_bytes", "kept_bytes", "dst_bytes")]


class rs_timing(C.Structure):
    _fields_ = [("ms", C.c_float), ("tiles", C.c_uint64), ("bytes", C.c_uint64), ("launches", C.c_uint64),
                ("read_bytes", C.c_uint64), ("main_ms", C.c_float)]


class rs_cell_binding(C.Structure):
    _fields_ = [("gpu", C.c_int32), ("arena", C.c_int32), ("offset", C.c_uint64), ("bytes", C.c_uint64)]


P = C.c_void_p
I32P = C.POINTER(C.c_int32)
U64P = C.POINTER(C.c_uint64)

# name: (restype, argtypes)
SIGNATURES = {
    "rs_last_error": (C.c_char_p, []),
    "rs_errc_name": (C.c_char_p, [C.c_int]),
    "rs_errc_count": (C.c_int, []),
    "rs_fnv1a64": (C.c_uint64, [P, C.c_uint64]),
    "rs_payload_seed": (C.c_uint64, [C.c_char_p]),
    "rs_build_info": (C.c_char_p, []),
    "rs_range_parse": (C.c_int, [C.c_char_p, C.POINTER(rs_range)]),
    "rs_range_format": (C.c_int, [C.POINTER(rs_range), C.c_char_p, C.c_uint64]),
    "rs_grid_cells": (C.c_int, [C.c_int, U64P, I32P, U64P, C.c_int, C.POINTER(rs_range), C.POINTER(C.c_int)]),
    "rs_grid_refine": (C.c_int, [C.c_int, I32P, U64P, C.c_int, I32P, U64P, I32P, U64P]),
    "rs_even_split": (C.c_int, [C.c_int, U64P, C.c_int, C.c_uint64, I32P, U64P]),
    "rs_grid_cell": (C.c_int, [C.c_int, U64P, I32P, U64P, C.c_uint64, C.POINTER(rs_range)]),
    "rs_grid_cell_index_of": (C.c_int, [C.c_int, U64P, I32P, U64P, C.POINTER(rs_range), U64P]),
    "rs_range_offset_by": (C.c_int, [C.POINTER(rs_range), C.POINTER(rs_range), C.POINTER(rs_range)]),
    "rs_range_valid_for": (C.c_int, [C.POINTER(rs_range), C.c_int, U64P, I32P]),
    "rs_rangespec_resolve": (C.c_int, [C.c_char_p, C.c_int, U64P, C.POINTER(rs_range)]),
    "rs_dtype_from_name": (C.c_int, [C.c_char_p, I32P]),
    "rs_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "rs_init": (C.c_int, [C.c_int, C.c_int, I32P, I32P, C.POINTER(P)]),
    "rs_destroy": (None, [P]),
    "rs_malloc": (C.c_int, [P, C.c_int, C.c_uint64, C.POINTER(P)]),
    "rs_free": (C.c_int, [P, C.c_int, P]),
    "rs_host_alloc": (C.c_int, [C.c_uint64, C.POINTER(P)]),
    "rs_host_free": (C.c_int, [P]),
    "rs_memcpy_htod": (C.c_int, [P, C.c_int, P, P, C.c_uint64]),
    "rs_memcpy_dtoh": (C.c_int, [P, C.c_int, P, P, C.c_uint64]),
    "rs_memset": (C.c_int, [P, C.c_int, P, C.c_int, C.c_uint64]),
    "rs_sync": (C.c_int, [P, C.c_int]),
    "rs_ipc_get_handle": (C.c_int, [P, C.c_int, P, P]),
    "rs_ipc_open_handle": (C.c_int, [P, C.c_int, P, C.POINTER(P)]),
    "rs_ipc_close_handle": (C.c_int, [P, C.c_int, P]),
    "rs_slice": (C.c_int, [P, C.c_int, C.POINTER(rs_tensor), C.POINTER(rs_range), P]),
    "rs_merge": (C.c_int, [P, C.c_int, C.c_int, C.POINTER(rs_range), C.POINTER(rs_tensor), C.c_int, U64P, P]),
    "rs_slice_host": (C.c_int, [P, C.c_int, C.POINTER(rs_tensor), C.POINTER(rs_range), P]),
    "rs_broadcast": (C.c_int, [P, C.c_int, P, C.c_int, C.POINTER(C.c_void_p), C.c_uint64, P]),
    "rs_merge_host": (C.c_int, [P, C.c_int, C.c_int, C.POINTER(rs_range), C.POINTER(rs_tensor), C.c_int, U64P, P]),
    "rs_catalog_create": (C.c_int, [C.POINTER(P)]),
    "rs_catalog_gpt": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.POINTER(P)]),
    "rs_catalog_add": (C.c_int, [P, C.c_char_p, C.c_int, C.c_int, U64P, C.c_int, C.c_int]),
    "rs_catalog_size": (C.c_int, [P]),
    "rs_catalog_get": (C.c_int, [P, C.c_int, C.c_char_p, C.c_int, I32P, I32P, U64P, I32P, I32P]),
    "rs_catalog_bytes": (C.c_uint64, [P]),
    "rs_catalog_destroy": (None, [P]),
    "rs_build_strategy": (C.c_int, [P, C.c_int, C.POINTER(rs_device), C.c_int, C.c_int, C.c_int, C.POINTER(P)]),
    "rs_ptc_destroy": (None, [P]),
    "rs_ptc_set_alpha": (C.c_int, [P, C.c_int, C.c_int, C.POINTER(rs_device)]),
    "rs_ptc_set_sigma": (C.c_int, [P, C.c_int, C.c_int, I32P, U64P]),
    "rs_validate": (C.c_int, [P, C.c_char_p, C.c_uint64, C.POINTER(C.c_int)]),
    "rs_hosted_subtensors": (C.c_int, [P, rs_device, C.c_int, I32P, C.POINTER(rs_range), C.POINTER(C.c_int)]),
    "rs_ptc_devices": (C.c_int, [P, C.c_int, C.POINTER(rs_device), C.POINTER(C.c_int)]),
    "rs_ptc_cell": (C.c_int, [P, C.c_int, C.c_int, C.POINTER(rs_range)]),
    "rs_ptc_cell_count": (C.c_int, [P, C.c_int, C.POINTER(C.c_int)]),
    "rs_parse_parallel_config": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(rs_device), C.POINTER(P)]),
    "rs_serialize_parallel_config": (C.c_int64, [P, C.c_char_p, C.c_int64]),
    "rs_generate_plan": (C.c_int, [P, P, C.POINTER(P)]),
    "rs_recover": (C.c_int, [P, C.c_int, C.POINTER(rs_device), P, C.POINTER(P)]),
    "rs_plan_destroy": (None, [P]),
    "rs_plan_get_stats": (C.c_int, [P, C.POINTER(rs_plan_stats)]),
    "rs_plan_cost": (C.c_int, [P, C.c_int, C.POINTER(rs_device), U64P, U64P, C.POINTER(C.c_int)]),
    "rs_plan_text": (C.c_int64, [P, C.c_char_p, C.c_int64]),
    "rs_plan_cost_central": (C.c_int, [P, rs_device, C.c_int, C.POINTER(rs_device), U64P, U64P, C.POINTER(C.c_int)]),
    "rs_choose_source": (C.c_int, [C.c_int, C.POINTER(rs_device), U64P, rs_device, C.POINTER(rs_device)]),
    "rs_executor_create": (C.c_int, [P, P, I32P, I32P, C.c_uint64, C.POINTER(P)]),
    "rs_executor_create_window": (C.c_int, [P, P, I32P, I32P, C.c_uint64, C.c_uint32, C.c_uint32, C.POINTER(P)]),
    "rs_executor_create_central": (C.c_int, [P, P, I32P, I32P, C.c_uint64, C.c_int, C.POINTER(P)]),
    "rs_executor_staging_bytes": (C.c_int, [P, U64P]),
    "rs_executor_destroy": (None, [P]),
    "rs_executor_arena_bytes": (C.c_int, [P, C.c_int, U64P, U64P]),
    "rs_executor_bind": (C.c_int, [P, C.c_int, P, P]),
    "rs_executor_prepare": (C.c_int, [P]),
    "rs_executor_run": (C.c_int, [P]),
    "rs_executor_wait": (C.c_int, [P, C.c_int, C.POINTER(rs_timing), C.POINTER(C.c_int)]),
    "rs_executor_run_host": (C.c_int, [P, C.c_int, P, P, C.POINTER(rs_timing)]),
    "rs_executor_run_host_flags": (C.c_int, [P, C.c_int, P, P, C.c_uint, C.POINTER(rs_timing)]),
    "rs_executor_host_upload_bytes": (C.c_int, [P, C.c_int, C.c_uint, C.POINTER(C.c_uint64)]),
    "rs_executor_host_phase": (C.c_int, [P, C.c_int, C.c_int, P]),
    "rs_executor_host_elapsed": (C.c_int, [P, C.c_int, C.POINTER(C.c_float)]),
    "rs_executor_world_ms": (C.c_int, [P, C.POINTER(C.c_float)]),
    "rs_executor_run_host_world": (C.c_int, [P, C.c_int, C.POINTER(P), C.POINTER(P), C.POINTER(C.c_float)]),
    "rs_executor_digests": (C.c_int, [P, C.c_int, C.c_int, C.c_int, I32P, U64P, I32P, C.POINTER(C.c_int)]),
    "rs_ipc_event_create": (C.c_int, [P, C.c_int, P, C.POINTER(P)]),
    "rs_ipc_event_open": (C.c_int, [P, C.c_int, P, C.POINTER(P)]),
    "rs_timing_event_create": (C.c_int, [P, C.c_int, C.POINTER(P)]),
    "rs_event_record": (C.c_int, [P, C.c_int, P]),
    "rs_event_wait": (C.c_int, [P, C.c_int, P]),
    "rs_event_elapsed": (C.c_int, [P, P, C.POINTER(C.c_float)]),
    "rs_event_destroy": (None, [P]),
    "rs_executor_fill_sources": (C.c_int, [P]),
    "rs_executor_verify": (C.c_int, [P, U64P]),
    "rs_executor_src_cells": (C.c_int, [P, C.c_int, C.POINTER(rs_cell_binding), C.POINTER(C.c_int)]),
    "rs_executor_dst_cells": (C.c_int, [P, C.c_int, C.POINTER(rs_cell_binding), I32P, I32P, I32P,
                                        C.POINTER(C.c_int)]),
    "rs_executor_tiles": (C.c_int, [P, C.c_int, U64P, U64P]),
    "rs_executor_read_bytes": (C.c_int, [P, C.c_int, U64P]),
    "rs_executor_bytes_to": (C.c_int, [P, C.c_int, C.c_int, U64P]),
    "rs_ptx_encoded_size": (C.c_int, [C.c_int, C.c_int, U64P, U64P]),
    "rs_ptx_encode_header": (C.c_int, [C.c_int, C.c_int, U64P, P, C.c_uint64, U64P]),
    "rs_ptx_decode_header": (C.c_int, [P, C.c_uint64, I32P, I32P, U64P, U64P]),
    "rs_checkpoint_save": (C.c_int, [P, C.c_int, C.c_char_p, U64P, U64P, C.POINTER(C.c_double)]),
    "rs_checkpoint_load": (C.c_int, [P, C.c_char_p, U64P, U64P, C.POINTER(C.c_double)]),
    "rs_shuffle_epoch": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, P]),
    "rs_repartition_count": (C.c_int, [C.c_uint64] * 5 + [U64P]),
    "rs_repartition_position": (C.c_int, [C.c_uint64] * 6 + [U64P]),
    "rs_locate_sample": (C.c_int, [C.c_uint64] * 6 + [P, P, P, U64P]),
    "rs_repartition_scratch_bytes": (C.c_int, [C.c_uint64, U64P]),
    "rs_dataset_index_pad": (C.c_int, [P, C.c_int, P, P, C.c_uint64, P]),
    "rs_dataset_index_upload": (C.c_int, [P, C.c_int, P, P, C.c_uint64, P, P, P, P]),
    "rs_repartition_to_host": (C.c_int, [P, C.c_int, C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                         C.c_void_p, P, C.c_void_p, P]),
    "rs_shuffle_scratch_bytes": (C.c_int, [C.c_uint64, U64P]),
    "rs_shuffle_epoch_device": (C.c_int, [P, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, P, P,
                                          C.POINTER(rs_timing)]),
    "rs_repartition": (C.c_int, [P, C.c_int, C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p,
                                 P, C.POINTER(rs_timing)]),
    "rs_repartition_gather_probe": (C.c_int, [P, C.c_int, C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                              C.c_int, C.POINTER(rs_timing)]),
    "rs_repartition_batch": (C.c_int, [P, C.c_int, C.c_void_p, C.c_uint64, C.c_void_p, C.c_int, C.c_void_p,
                                       C.POINTER(rs_timing)]),
}


class rs_dataset_index(C.Structure):
    _fields_ = [("perm", C.c_void_p), ("samples", C.c_void_p), ("file_class", C.c_void_p), ("n", C.c_uint64),
                ("entry_bytes", C.c_uint64)]


class rs_partition_host(C.Structure):
    _fields_ = [("pos", C.c_void_p), ("ent", C.c_void_p), ("boff", C.c_void_p), ("queue", C.c_void_p * 3),
                ("qcount", C.c_void_p)]


class rs_partition_out(C.Structure):
    _fields_ = [("pos", C.c_void_p), ("ent", C.c_void_p), ("boff", C.c_void_p), ("queue", C.c_void_p * 3),
                ("qcount", C.c_void_p)]


class rs_repartition_job(C.Structure):
    _fields_ = [("at_step", C.c_uint64), ("new_dp", C.c_uint64), ("rank", C.c_uint64), ("file_class", C.c_void_p),
                ("out", rs_partition_out), ("scratch", C.c_void_p)]


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -m paper_2312_05181_b200.build` "
            "(the reshard path has no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib
