"""TEST INFRASTRUCTURE ONLY -- Python loader for the CPU parity oracle.

Two checkers, both CPU:
  * ``port``: oracle/liboracle.so, the plain-C restatement (hull_oracle.c);
  * ``ref``:  oracle/_ref/libhull2d_ref.so, the unmodified reference headers
    behind a C-ABI (ref_driver.cpp). Built here from /root/reference; the
    prebuilt .so travels to the GPU box (git-ignored, not gpurun-ignored).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) may import this package. The product never does.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_PATH = HERE / "liboracle.so"
REF_PATH = HERE / "_ref" / "libhull2d_ref.so"


class oc_config(C.Structure):
    _fields_ = [("chunk_count", C.c_uint64), ("enable_round1", C.c_int32),
                ("enable_round2", C.c_int32), ("chunked", C.c_int32), ("reserved", C.c_int32)]


class oc_stats(C.Structure):
    _fields_ = [("n_input", C.c_uint64), ("n_after_round1", C.c_uint64),
                ("n_after_round2", C.c_uint64), ("hull_size", C.c_uint64),
                ("t_round1_ms", C.c_double), ("t_annotate_ms", C.c_double),
                ("t_sort_ms", C.c_double), ("t_round2_ms", C.c_double),
                ("t_finalize_ms", C.c_double), ("t_total_ms", C.c_double)]


class oc_trace(C.Structure):
    _fields_ = [("quad", C.c_uint64 * 4), ("anchor", C.c_uint64),
                ("r1_idx", C.POINTER(C.c_uint64)), ("sorted_idx", C.POINTER(C.c_uint64)),
                ("sorted_len", C.c_uint64), ("longest", C.c_uint64),
                ("r2_flags", C.POINTER(C.c_uint8)), ("r2_idx", C.POINTER(C.c_uint64))]


_DP = C.POINTER(C.c_double)
_U64P = C.POINTER(C.c_uint64)
_U8P = C.POINTER(C.c_uint8)

_port = None
_ref = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def port() -> C.CDLL:
    global _port
    if _port is None:
        if not PORT_PATH.exists():
            build()
        lib = C.CDLL(str(PORT_PATH))
        lib.oc_full_pipeline.restype = C.c_int
        lib.oc_full_pipeline.argtypes = [_DP, _DP, C.c_uint64, C.POINTER(oc_config), _U64P,
                                         C.c_uint64, _U64P, C.POINTER(oc_stats),
                                         C.POINTER(oc_trace)]
        lib.oc_find_extremes.argtypes = [_DP, _DP, C.c_uint64, _U64P]
        lib.oc_select_anchor.restype = C.c_uint64
        lib.oc_select_anchor.argtypes = [_DP, _DP, C.c_uint64]
        lib.oc_classify_quad.argtypes = [_DP, _DP, C.c_uint64, _U64P, _U8P]
        lib.oc_orient.restype = C.c_int
        lib.oc_orient.argtypes = [C.c_double] * 6
        lib.oc_atan2.restype = C.c_double
        lib.oc_atan2.argtypes = [C.c_double, C.c_double]
        lib.oc_atan2_array.argtypes = [_DP, _DP, _DP, C.c_uint64]
        lib.oc_monotone_chain.argtypes = [_DP, _DP, C.c_uint64, _U64P, C.c_uint64, _U64P]
        _port = lib
    return _port


def ref_available() -> bool:
    return REF_PATH.exists()


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not REF_PATH.exists():
            raise FileNotFoundError(f"{REF_PATH} not built (needs /root/reference at build time)")
        lib = C.CDLL(str(REF_PATH))
        lib.ref_full_pipeline.restype = C.c_int
        lib.ref_full_pipeline.argtypes = [_DP, _DP, C.c_uint64, C.c_uint64, C.c_int, C.c_int,
                                          C.c_int, _U64P, C.c_uint64, _U64P,
                                          C.POINTER(oc_stats)]
        lib.ref_monotone_chain.argtypes = [_DP, _DP, C.c_uint64, _U64P, C.c_uint64, _U64P]
        lib.ref_find_extremes.argtypes = [_DP, _DP, C.c_uint64, _U64P]
        lib.ref_classify.argtypes = [_DP, _DP, C.c_uint64, _U8P]
        lib.ref_sorted_buffer.argtypes = [_DP, _DP, C.c_uint64, _U64P, _DP, _DP, _U64P]
        lib.ref_discard_flags.argtypes = [_DP, _DP, C.c_uint64, C.c_uint64, C.c_int, _U8P, _U64P]
        lib.ref_generate.argtypes = [C.c_int, C.c_uint64, C.c_uint64, _DP, _DP]
        lib.ref_load.restype = C.c_int
        lib.ref_load.argtypes = [C.c_char_p, C.c_int, _DP, _DP, C.c_uint64, _U64P, C.c_char_p,
                                 C.c_uint64]
        _ref = lib
    return _ref


def _d(a: np.ndarray):
    return a.ctypes.data_as(_DP)


def _u(a: np.ndarray):
    return a.ctypes.data_as(_U64P)


def _soa(xs, ys):
    return (np.ascontiguousarray(xs, dtype=np.float64), np.ascontiguousarray(ys, dtype=np.float64))


def stats_dict(s: oc_stats) -> dict:
    return {f: getattr(s, f) for f, _ in oc_stats._fields_}


def full_pipeline(xs, ys, chunk_count=1024, enable_round1=True, enable_round2=True, chunked=True,
                  trace=False, impl="port"):
    """Returns (hull indices uint64, stats dict[, trace dict]). impl: 'port' | 'ref'."""
    xs, ys = _soa(xs, ys)
    n = xs.shape[0]
    out = np.empty(max(n, 1), np.uint64)
    out_len = C.c_uint64()
    st = oc_stats()
    if impl == "ref":
        rc = ref().ref_full_pipeline(_d(xs), _d(ys), n, chunk_count, int(enable_round1),
                                     int(enable_round2), int(chunked), _u(out), out.shape[0],
                                     C.byref(out_len), C.byref(st))
        if rc:
            raise RuntimeError(f"reference full_pipeline status {rc}")
        return out[: out_len.value].copy(), stats_dict(st)
    cfg = oc_config(chunk_count, int(enable_round1), int(enable_round2), int(chunked), 0)
    tr = None
    bufs = {}
    if trace:
        bufs = {"r1_idx": np.empty(max(n, 1), np.uint64),
                "sorted_idx": np.empty(max(n, 1), np.uint64),
                "r2_flags": np.empty(max(n, 1), np.uint8),
                "r2_idx": np.empty(max(n, 1), np.uint64)}
        tr = oc_trace()
        tr.r1_idx = _u(bufs["r1_idx"])
        tr.sorted_idx = _u(bufs["sorted_idx"])
        tr.r2_flags = bufs["r2_flags"].ctypes.data_as(_U8P)
        tr.r2_idx = _u(bufs["r2_idx"])
    rc = port().oc_full_pipeline(_d(xs), _d(ys), n, C.byref(cfg), _u(out), out.shape[0],
                                 C.byref(out_len), C.byref(st), C.byref(tr) if tr else None)
    if rc:
        raise RuntimeError(f"oracle full_pipeline status {rc}")
    hull_idx = out[: out_len.value].copy()
    sd = stats_dict(st)
    if not trace:
        return hull_idx, sd
    m = tr.sorted_len
    t = {"quad": list(tr.quad), "anchor": tr.anchor, "longest": tr.longest,
         "r1_idx": bufs["r1_idx"][: sd["n_after_round1"]].copy(),
         "sorted_idx": bufs["sorted_idx"][:m].copy(),
         "r2_flags": bufs["r2_flags"][:m].copy() if enable_round2 and m >= 2 else None,
         "r2_idx": bufs["r2_idx"][: sd["n_after_round2"]].copy()}
    return hull_idx, sd, t


def monotone_chain(xs, ys, impl="port") -> np.ndarray:
    xs, ys = _soa(xs, ys)
    n = xs.shape[0]
    out = np.empty(max(n, 1) + 1, np.uint64)
    k = C.c_uint64()
    lib = ref() if impl == "ref" else port()
    fn = lib.ref_monotone_chain if impl == "ref" else lib.oc_monotone_chain
    rc = fn(_d(xs), _d(ys), n, _u(out), out.shape[0], C.byref(k))
    if rc:
        raise RuntimeError(f"monotone_chain status {rc}")
    return out[: k.value].copy()


def ref_sorted_buffer(xs, ys):
    xs, ys = _soa(xs, ys)
    n = xs.shape[0]
    idx = np.empty(max(n, 1), np.uint64)
    ang = np.empty(max(n, 1))
    d2 = np.empty(max(n, 1))
    m = C.c_uint64()
    rc = ref().ref_sorted_buffer(_d(xs), _d(ys), n, _u(idx), _d(ang), _d(d2), C.byref(m))
    if rc:
        raise RuntimeError(f"ref_sorted_buffer status {rc}")
    k = m.value
    return idx[:k].copy(), ang[:k].copy(), d2[:k].copy()


def ref_discard_flags(xs, ys, chunk_count=1024, chunked=True):
    xs, ys = _soa(xs, ys)
    n = xs.shape[0]
    flags = np.empty(max(n, 1), np.uint8)
    l = C.c_uint64()
    rc = ref().ref_discard_flags(_d(xs), _d(ys), n, chunk_count, int(chunked),
                                 flags.ctypes.data_as(_U8P), C.byref(l))
    if rc:
        raise RuntimeError(f"ref_discard_flags status {rc}")
    return flags, l.value


def ref_generate(kind: int, n: int, seed: int):
    xs = np.empty(n)
    ys = np.empty(n)
    rc = ref().ref_generate(kind, n, seed, _d(xs), _d(ys))
    if rc:
        raise RuntimeError("ref_generate failed")
    return xs, ys


def ref_load(path, obj=False, cap=1 << 20):
    """The reference's load_points / load_obj_projected: (code, xs, ys, message);
    code 0 ok, 1 ParseError, 2 IoError, 3 EmptyInput."""
    xs = np.empty(cap)
    ys = np.empty(cap)
    n = C.c_uint64()
    msg = C.create_string_buffer(512)
    rc = ref().ref_load(str(path).encode(), int(obj), _d(xs), _d(ys), cap, C.byref(n), msg, 512)
    k = min(n.value, cap)
    return rc, xs[:k].copy(), ys[:k].copy(), msg.value.decode()


def find_extremes(xs, ys) -> list[int]:
    xs, ys = _soa(xs, ys)
    q = np.zeros(4, np.uint64)
    rc = port().oc_find_extremes(_d(xs), _d(ys), xs.shape[0], _u(q))
    if rc:
        raise RuntimeError("EmptyInput")
    return [int(v) for v in q]


def select_anchor(xs, ys) -> int:
    xs, ys = _soa(xs, ys)
    return int(port().oc_select_anchor(_d(xs), _d(ys), xs.shape[0]))


def classify_quad(xs, ys, quad) -> np.ndarray:
    xs, ys = _soa(xs, ys)
    q = np.asarray(quad, np.uint64)
    f = np.empty(xs.shape[0], np.uint8)
    port().oc_classify_quad(_d(xs), _d(ys), xs.shape[0], _u(q), f.ctypes.data_as(_U8P))
    return f


def orient(a, b, c) -> int:
    return int(port().oc_orient(a[0], a[1], b[0], b[1], c[0], c[1]))


def atan2(y: float, x: float) -> float:
    return float(port().oc_atan2(y, x))


def atan2_array(y, x) -> np.ndarray:
    """Host libm atan2 (the reference's std::atan2) elementwise."""
    y, x = _soa(y, x)
    out = np.empty_like(y)
    port().oc_atan2_array(_d(y), _d(x), _d(out), y.shape[0])
    return out
