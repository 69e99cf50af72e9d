"""ctypes binding of the in-tree native library (include/gscan.h).

The library is the product: there is no Python or CPU fallback. If it is
missing or no CUDA device is visible, calls raise ``NativeUnavailable``.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "_lib" / "libgscan.so"
if os.environ.get("GSCAN_LIB"):  # development: an alternative build (tools/micro)
    LIB_PATH = Path(os.environ["GSCAN_LIB"])

GSCAN_OK = 0
GSCAN_E_EMPTY_INPUT = 1
GSCAN_E_ZERO_CHUNKS = 2
GSCAN_E_CAPACITY = 3
GSCAN_E_CUDA = 4
GSCAN_E_INVALID = 5
GSCAN_E_TOO_LARGE = 6
GSCAN_E_NO_DEVICE = 7
GSCAN_E_INTERNAL = 8
GSCAN_E_IO = 9
GSCAN_E_PARSE = 10
GSCAN_E_NCCL = 11
FMT_XY, FMT_OBJ, FMT_SOA = 0, 1, 2

GEN_SQUARE, GEN_DISK, GEN_CIRCLE, GEN_COLLINEAR = 0, 1, 2, 3

DEBUG_FORCE_JUNCTION = 1 << 0
DEBUG_FORCE_SEQUENTIAL = 1 << 1
DEBUG_CORRUPT_CANDIDATE = 1 << 2
DEBUG_FORCE_FALLBACK = 1 << 3
DEBUG_FORCE_PREFIX = 1 << 4
DEBUG_FULL_SORT = 1 << 5
DEBUG_SPARSE_DROP = 1 << 6
DEBUG_SPARSE_VERIFY = 1 << 7


class NativeUnavailable(RuntimeError):
    """libgscan.so is not built or cannot run here (no CUDA device)."""


class gscan_config(C.Structure):
    _fields_ = [("chunk_count", C.c_uint64), ("enable_round1", C.c_int32),
                ("enable_round2", C.c_int32), ("chunked", C.c_int32), ("reserved", C.c_int32)]


class gscan_stats(C.Structure):
    _fields_ = [("n_input", C.c_uint64), ("n_after_round1", C.c_uint64),
                ("n_after_round2", C.c_uint64), ("hull_size", C.c_uint64),
                ("t_round1_ms", C.c_double), ("t_annotate_ms", C.c_double),
                ("t_sort_ms", C.c_double), ("t_round2_ms", C.c_double),
                ("t_finalize_ms", C.c_double), ("t_total_ms", C.c_double)]


class gscan_extremes(C.Structure):
    _fields_ = [("idx", C.c_uint64 * 5), ("x", C.c_double * 5), ("y", C.c_double * 5)]


class gscan_dist_bufs(C.Structure):
    _fields_ = [("rec", C.c_void_p), ("recs", C.c_void_p), ("ext", C.c_void_p),
                ("cells", C.c_void_p), ("hist", C.c_void_p), ("phimax", C.c_void_p),
                ("pref", C.c_void_p), ("part_counts", C.c_void_p), ("parted", C.c_void_p),
                ("rlo", C.c_void_p), ("rx", C.c_void_p), ("ry", C.c_void_p), ("stream", C.c_void_p),
                ("rec_len", C.c_uint64), ("max_ranks", C.c_uint64), ("buckets", C.c_uint64),
                ("cells_n", C.c_uint64), ("parts", C.c_uint64)]


# sparse-path sizes the sharded phases exchange (csrc/sparse.cuh)
SP_CELLS = 2048
SP_BUCKETS = 48 * 1024
SP_PARTS = 2048
SP_FAIL_TIE, SP_FAIL_FEW, SP_FAIL_MANY = 1, 128, 256
SP_FAIL_CAP = 32

# Every symbol include/gscan.h declares, with its ctypes signature.
_P = C.c_void_p
_U64 = C.c_uint64
_U64P = C.POINTER(C.c_uint64)
_DP = C.POINTER(C.c_double)
SIGNATURES = {
    "gscan_config_default": (None, [C.POINTER(gscan_config)]),
    "gscan_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "gscan_destroy": (C.c_int, [_P]),
    "gscan_reserve": (C.c_int, [_P, _U64]),
    "gscan_set_stream": (C.c_int, [_P, _P]),
    "gscan_hull_f64": (C.c_int, [_P, _DP, _DP, _U64, C.POINTER(gscan_config), _U64P, _U64, _U64P,
                                 C.POINTER(gscan_stats)]),
    "gscan_hull_f64_device": (C.c_int, [_P, _P, _P, _U64, C.POINTER(gscan_config), _P, _U64,
                                        _U64P, C.POINTER(gscan_stats)]),
    "gscan_hull": (C.c_int, [_DP, _DP, _U64, _U64P, _U64, _U64P]),
    "gscan_stage_extremes": (C.c_int, [_P, _P, _P, _U64, _U64P]),
    "gscan_stage_round1": (C.c_int, [_P, _P, _P, _U64, _P, _U64P]),
    "gscan_stage_sorted": (C.c_int, [_P, _P, _P, _U64, _P, _U64P]),
    "gscan_stage_discard": (C.c_int, [_P, _P, _P, _U64, _U64, C.c_int, _P, _U64P, _U64P]),
    "gscan_device_atan2": (C.c_int, [_P, _P, _P, _P, _U64]),
    "gscan_shard_extremes": (C.c_int, [_P, _P, _P, _U64, C.POINTER(gscan_extremes)]),
    "gscan_shard_round1": (C.c_int, [_P, _P, _P, _U64, C.POINTER(gscan_extremes), _P, _U64P]),
    "gscan_dist_enq_begin": (C.c_int, [_P, _P, _P, _U64, _U64, C.POINTER(gscan_config)]),
    "gscan_dist_buffers": (C.c_int, [_P, C.POINTER(gscan_dist_bufs)]),
    "gscan_dist_enq_sample": (C.c_int, [_P, C.c_uint32]),
    "gscan_dist_enq_f2": (C.c_int, [_P]),
    "gscan_dist_enq_plan": (C.c_int, [_P, C.c_uint32, _U64]),
    "gscan_dist_enq_f3": (C.c_int, [_P, C.c_uint32]),
    "gscan_dist_enq_dup_local": (C.c_int, [_P, C.c_uint32]),
    "gscan_dist_enq_dup_check": (C.c_int, [_P, _P, _U64, _P, C.c_uint32]),
    "gscan_dist_enq_export": (C.c_int, [_P, C.c_int, _P, _P, _P, _P]),
    "gscan_dist_enq_slices": (C.c_int, [_P, _P, _P, _U64, _P, _P, _U64]),
    "gscan_dist_enq_cand": (C.c_int, [_P]),
    "gscan_dist_root_finish": (C.c_int, [_P, _P, _P, _U64, _U64, _P, _U64, _P, _U64, _U64P, _U64P,
                                         C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
    "gscan_dist_enq_verify": (C.c_int, [_P, _P, _P, _P]),
    "gscan_shard_keys": (C.c_int, [_P, _P, _P, _P, _U64, C.POINTER(gscan_extremes), _P]),
    "gscan_hull_sorted": (C.c_int, [_P, _P, _P, _U64, C.POINTER(gscan_config), _P, _U64, _U64P,
                                    _U64P]),
    "gscan_status_string": (C.c_char_p, [C.c_int]),
    "gscan_last_error": (C.c_char_p, [_P]),
    "gscan_last_launch_count": (_U64, [_P]),
    "gscan_set_profiling": (C.c_int, [_P, C.c_int]),
    "gscan_set_debug": (C.c_int, [_P, C.c_uint32]),
    "gscan_last_graham_info": (C.c_int, [_P, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
    "gscan_last_sparse_info": (C.c_int, [_P, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                         C.POINTER(C.c_uint32)]),
    "gscan_last_kernel_times": (C.c_int, [_P, C.POINTER(C.c_char_p), _DP, C.c_int]),
    "gscan_generate": (C.c_int, [C.c_int, _U64, _U64, _DP, _DP]),
    "gscan_generate_grid": (C.c_int, [_U64, _U64, C.c_int, C.c_int, _DP, _DP]),
    "gscan_generate_square_device": (C.c_int, [_P, _U64, _U64, _U64, _P, _P]),
    "gscan_mt64_jump_check": (C.c_int, [_U64, _U64]),
    "gscan_load": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(_DP), C.POINTER(_DP), _U64P]),
    "gscan_soa_count": (C.c_int, [C.c_char_p, _U64P]),
    "gscan_soa_read": (C.c_int, [C.c_char_p, _DP, _DP, _U64]),
    "gscan_save_soa": (C.c_int, [C.c_char_p, _DP, _DP, _U64]),
    "gscan_free": (None, [C.c_void_p]),
    "gscan_io_error": (C.c_char_p, []),
}

_lib = None


def load(path: str | os.PathLike | None = None) -> C.CDLL:
    """Load libgscan.so (once) and attach signatures. Raises NativeUnavailable."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise NativeUnavailable(
            f"{p} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def status_string(code: int) -> str:
    return load().gscan_status_string(code).decode()
