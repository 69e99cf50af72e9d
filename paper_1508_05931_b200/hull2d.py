"""Host-side mirror of the reference ``hull2d`` pipeline interface.

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/include/hull2d/pipeline.hpp:19-51,72; errors.hpp:9-49),
so parity tests read like the reference's own tests:

    result = full_pipeline(points, PipelineConfig(chunk_count=7))
    result.hull.vertices      # (k, 2) float64, CCW from the anchor
    result.hull.indices       # (k,) uint64 first-occurrence input indices (north star)
    result.stats.n_after_round1 ...

Every call runs the sm_100a kernels in ``libgscan.so``; nothing here computes
a hull on the CPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N


# ---- errors (errors.hpp:9-49) ----
class Error(RuntimeError):
    pass


class EmptyInput(Error):
    pass


class LengthMismatch(Error):
    pass


class CoincidentWithAnchor(Error):
    pass


class TooFewPoints(Error):
    pass


class IndexOutOfRange(Error):
    pass


class ZeroChunks(Error):
    pass


class TooLarge(Error):
    pass


class DeviceError(Error):
    """CUDA runtime failure inside the native library."""


class IoError(Error):
    """errors.hpp IoError: a file cannot be opened or read (datagen.hpp loaders)."""


class ParseError(Error):
    """errors.hpp ParseError: a malformed line (the message names its number)."""


class CollectiveError(Error):
    """A collective of the sharded path failed (GSCAN_E_NCCL)."""


_STATUS_EXC = {
    N.GSCAN_E_EMPTY_INPUT: EmptyInput,
    N.GSCAN_E_ZERO_CHUNKS: ZeroChunks,
    N.GSCAN_E_TOO_LARGE: TooLarge,
    N.GSCAN_E_CUDA: DeviceError,
    N.GSCAN_E_INTERNAL: DeviceError,
    N.GSCAN_E_INVALID: ValueError,
    N.GSCAN_E_NO_DEVICE: N.NativeUnavailable,
    N.GSCAN_E_IO: IoError,
    N.GSCAN_E_PARSE: ParseError,
    N.GSCAN_E_NCCL: CollectiveError,
}


# ---- value types (pipeline.hpp:19-51) ----
@dataclass
class PipelineConfig:
    chunk_count: int = 1024
    enable_round1: bool = True
    enable_round2: bool = True
    chunked: bool = True

    def _c(self) -> N.gscan_config:
        if self.chunk_count < 0:
            raise ValueError("chunk_count must be non-negative")
        return N.gscan_config(int(self.chunk_count), int(bool(self.enable_round1)),
                              int(bool(self.enable_round2)), int(bool(self.chunked)), 0)


@dataclass
class StageStats:
    n_input: int = 0
    n_after_round1: int = 0
    n_after_round2: int = 0
    hull_size: int = 0
    t_round1_ms: float = 0.0
    t_annotate_ms: float = 0.0
    t_sort_ms: float = 0.0
    t_round2_ms: float = 0.0
    t_finalize_ms: float = 0.0
    t_total_ms: float = 0.0

    @classmethod
    def _from_c(cls, s: N.gscan_stats) -> "StageStats":
        return cls(*(getattr(s, f) for f, _ in N.gscan_stats._fields_))


@dataclass
class Hull:
    vertices: np.ndarray  # (k, 2) float64
    indices: np.ndarray   # (k,) uint64, first occurrence in the input

    def size(self) -> int:
        return int(self.indices.shape[0])

    def __len__(self) -> int:
        return self.size()


@dataclass
class PipelineResult:
    hull: Hull
    stats: StageStats = field(default_factory=StageStats)


def _as_soa(points, ys=None) -> tuple[np.ndarray, np.ndarray]:
    if ys is not None:
        xs = np.ascontiguousarray(points, dtype=np.float64).reshape(-1)
        ys = np.ascontiguousarray(ys, dtype=np.float64).reshape(-1)
        if xs.shape != ys.shape:
            raise LengthMismatch("xs and ys differ in length")
        return xs, ys
    p = np.asarray(points, dtype=np.float64)
    if p.size == 0:
        return np.zeros(0), np.zeros(0)
    if p.ndim != 2 or p.shape[1] != 2:
        raise ValueError("points must be an (n, 2) array of (x, y)")
    return np.ascontiguousarray(p[:, 0]), np.ascontiguousarray(p[:, 1])


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class Engine:
    """One device handle (device scratch, stream). Not thread-safe per instance."""

    def __init__(self, device: int = -1):
        self._lib = N.load()
        h = C.c_void_p()
        rc = self._lib.gscan_create(int(device), C.byref(h))
        if rc != N.GSCAN_OK:
            raise _STATUS_EXC.get(rc, Error)(f"gscan_create: {N.status_string(rc)}")
        self._h = h

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.gscan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def _raise(self, rc: int, what: str):
        msg = self._lib.gscan_last_error(self._h).decode() or N.status_string(rc)
        raise _STATUS_EXC.get(rc, Error)(f"{what}: {msg}")

    def reserve(self, n: int) -> None:
        rc = self._lib.gscan_reserve(self._h, int(n))
        if rc:
            self._raise(rc, "reserve")

    def set_profiling(self, on: bool) -> None:
        self._lib.gscan_set_profiling(self._h, int(bool(on)))

    def kernel_times(self) -> list[tuple[str, float]]:
        cap = 256
        names = (C.c_char_p * cap)()
        ms = (C.c_double * cap)()
        k = self._lib.gscan_last_kernel_times(self._h, names, ms, cap)
        return [(names[i].decode(), ms[i]) for i in range(k)]

    def set_debug(self, flags: int) -> None:
        """Test hooks (include/gscan.h GSCAN_DEBUG_*)."""
        self._lib.gscan_set_debug(self._h, int(flags))

    def graham_info(self) -> tuple[int, int]:
        path = C.c_uint32()
        fails = C.c_uint32()
        self._lib.gscan_last_graham_info(self._h, C.byref(path), C.byref(fails))
        return path.value, fails.value

    def sparse_info(self) -> tuple[int, int, int]:
        """(used, fail_bits, n_walked) of the last call's sparse round-2 path."""
        u, f, w = C.c_uint32(), C.c_uint32(), C.c_uint32()
        self._lib.gscan_last_sparse_info(self._h, C.byref(u), C.byref(f), C.byref(w))
        return u.value, f.value, w.value

    def launch_count(self) -> int:
        return int(self._lib.gscan_last_launch_count(self._h))

    # -- full_pipeline (pipeline.hpp:72) on host arrays --
    def full_pipeline(self, points, cfg: PipelineConfig | None = None, ys=None) -> PipelineResult:
        xs, ys_ = _as_soa(points, ys)
        idx, st = self.hull_indices(xs, ys_, cfg)
        verts = np.stack([xs[idx], ys_[idx]], axis=1) if idx.size else np.zeros((0, 2))
        return PipelineResult(Hull(verts, idx), st)

    def hull_indices(self, xs: np.ndarray, ys: np.ndarray, cfg: PipelineConfig | None = None):
        xs = np.ascontiguousarray(xs, dtype=np.float64)
        ys = np.ascontiguousarray(ys, dtype=np.float64)
        if xs.shape != ys.shape:
            raise LengthMismatch("xs and ys differ in length")
        n = int(xs.shape[0])
        c = (cfg or PipelineConfig())._c()
        st = N.gscan_stats()
        out = np.empty(max(n, 1), dtype=np.uint64)
        out_len = C.c_uint64()
        rc = self._lib.gscan_hull_f64(self._h, _dptr(xs), _dptr(ys), n, C.byref(c),
                                      out.ctypes.data_as(C.POINTER(C.c_uint64)), out.shape[0],
                                      C.byref(out_len), C.byref(st))
        if rc:
            self._raise(rc, "full_pipeline")
        return out[: out_len.value].copy(), StageStats._from_c(st)

    def hull_ptr(self, xs_ptr: int, ys_ptr: int, n: int, out_ptr: int, out_cap: int,
                 cfg: PipelineConfig | None = None) -> tuple[int, StageStats]:
        """Host-pointer entry (e.g. pinned buffers); out_ptr receives uint64 indices."""
        c = (cfg or PipelineConfig())._c()
        st = N.gscan_stats()
        out_len = C.c_uint64()
        rc = self._lib.gscan_hull_f64(self._h, C.cast(xs_ptr, C.POINTER(C.c_double)),
                                      C.cast(ys_ptr, C.POINTER(C.c_double)), int(n), C.byref(c),
                                      C.cast(out_ptr, C.POINTER(C.c_uint64)), int(out_cap),
                                      C.byref(out_len), C.byref(st))
        if rc:
            self._raise(rc, "full_pipeline")
        return out_len.value, StageStats._from_c(st)

    def hull_device(self, d_xs: int, d_ys: int, n: int, d_out: int, out_cap: int,
                    cfg: PipelineConfig | None = None) -> tuple[int, StageStats]:
        """Device-pointer entry; d_out receives uint32 indices on the device."""
        cfg = cfg or PipelineConfig()
        key = (cfg.chunk_count, cfg.enable_round1, cfg.enable_round2, cfg.chunked)
        cache = getattr(self, "_dev_call", None)
        if cache is None or cache[0] != key:  # ctypes argument objects, reused per call
            cache = (key, cfg._c(), N.gscan_stats(), C.c_uint64())
            self._dev_call = cache
        _, c, st, out_len = cache
        rc = self._lib.gscan_hull_f64_device(self._h, d_xs, d_ys, n, C.byref(c), d_out, out_cap,
                                             C.byref(out_len), C.byref(st))
        if rc:
            self._raise(rc, "full_pipeline")
        return out_len.value, StageStats._from_c(st)

    def generate_square_device(self, seed: int, lo: int, hi: int, d_xs: int, d_ys: int) -> None:
        """Points [lo, hi) of gen_square(n >= hi, seed) (datagen.hpp:32-41) into
        device arrays, bit-identical to the host generator (mtgen.cuh)."""
        rc = self._lib.gscan_generate_square_device(self._h, int(seed), int(lo), int(hi),
                                                    C.c_void_p(d_xs), C.c_void_p(d_ys))
        if rc:
            self._raise(rc, "generate_square_device")

    # -- stage entry points (device pointers) --
    def stage_extremes(self, d_xs: int, d_ys: int, n: int) -> list[int]:
        out = (C.c_uint64 * 5)()
        rc = self._lib.gscan_stage_extremes(self._h, C.c_void_p(d_xs), C.c_void_p(d_ys), n, out)
        if rc:
            self._raise(rc, "find_extremes")
        return list(out)

    def stage_round1(self, d_xs: int, d_ys: int, n: int, d_out: int) -> int:
        k = C.c_uint64()
        rc = self._lib.gscan_stage_round1(self._h, C.c_void_p(d_xs), C.c_void_p(d_ys), n,
                                          C.c_void_p(d_out), C.byref(k))
        if rc:
            self._raise(rc, "round1")
        return k.value

    def stage_sorted(self, d_xs: int, d_ys: int, n: int, d_out: int) -> int:
        k = C.c_uint64()
        rc = self._lib.gscan_stage_sorted(self._h, C.c_void_p(d_xs), C.c_void_p(d_ys), n,
                                          C.c_void_p(d_out), C.byref(k))
        if rc:
            self._raise(rc, "sorted_buffer")
        return k.value

    def stage_discard(self, d_xs: int, d_ys: int, n: int, chunk_count: int, chunked: bool,
                      d_flags: int) -> tuple[int, int]:
        l = C.c_uint64()
        m = C.c_uint64()
        rc = self._lib.gscan_stage_discard(self._h, C.c_void_p(d_xs), C.c_void_p(d_ys), n,
                                           int(chunk_count), int(bool(chunked)),
                                           C.c_void_p(d_flags), C.byref(l), C.byref(m))
        if rc:
            self._raise(rc, "discard")
        return l.value, m.value

    def device_atan2(self, d_y: int, d_x: int, d_out: int, n: int) -> None:
        rc = self._lib.gscan_device_atan2(self._h, C.c_void_p(d_y), C.c_void_p(d_x),
                                          C.c_void_p(d_out), int(n))
        if rc:
            self._raise(rc, "atan2")


_default: Engine | None = None


def default_engine() -> Engine:
    global _default
    if _default is None:
        _default = Engine()
    return _default


def full_pipeline(points, cfg: PipelineConfig | None = None) -> PipelineResult:
    """hull2d::full_pipeline (pipeline.hpp:72) on the default device."""
    return default_engine().full_pipeline(points, cfg)


def hull(xs, ys) -> np.ndarray:
    """North-star entry: hull(xs, ys, n) -> ordered hull vertex indices (uint64)."""
    idx, _ = default_engine().hull_indices(np.asarray(xs, np.float64), np.asarray(ys, np.float64))
    return idx


# ---- harness helpers (host generators, bit-identical to datagen.hpp) ----
def generate(kind: str, n: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    kinds = {"square": N.GEN_SQUARE, "disk": N.GEN_DISK, "circle": N.GEN_CIRCLE,
             "collinear": N.GEN_COLLINEAR}
    xs = np.empty(n, np.float64)
    ys = np.empty(n, np.float64)
    rc = N.load().gscan_generate(kinds[kind], int(n), int(seed), _dptr(xs), _dptr(ys))
    if rc:
        raise ValueError(f"generate({kind}): {N.status_string(rc)}")
    return xs, ys


# ---- ingest (datagen.hpp:111-168 loaders, csrc/io.cpp) ----
_FMTS = {"xy": N.FMT_XY, "obj": N.FMT_OBJ, "soa": N.FMT_SOA}


def load_points(path, fmt: str = "xy") -> tuple[np.ndarray, np.ndarray]:
    """Points of a plain-XY text file (load_points), the vertex lines of an OBJ
    file (load_obj_projected) or a GSCANSOA binary file, as SoA float64 arrays.
    Raises IoError / ParseError / EmptyInput like the reference."""
    lib = N.load()
    xp, yp = C.POINTER(C.c_double)(), C.POINTER(C.c_double)()
    n = C.c_uint64()
    rc = lib.gscan_load(str(path).encode(), _FMTS[fmt], C.byref(xp), C.byref(yp), C.byref(n))
    if rc:
        raise _STATUS_EXC.get(rc, Error)(lib.gscan_io_error().decode())
    try:
        m = n.value
        xs = np.ctypeslib.as_array(xp, shape=(m,)).copy()
        ys = np.ctypeslib.as_array(yp, shape=(m,)).copy()
    finally:
        lib.gscan_free(C.cast(xp, C.c_void_p))
        lib.gscan_free(C.cast(yp, C.c_void_p))
    return xs, ys


def save_soa(path, xs, ys) -> None:
    """Write a GSCANSOA binary file (the device path's layout)."""
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    ys = np.ascontiguousarray(ys, dtype=np.float64)
    if xs.shape != ys.shape:
        raise LengthMismatch("xs and ys differ in length")
    lib = N.load()
    rc = lib.gscan_save_soa(str(path).encode(), _dptr(xs), _dptr(ys), xs.shape[0])
    if rc:
        raise _STATUS_EXC.get(rc, Error)(lib.gscan_io_error().decode())


def generate_grid(n: int, seed: int, lo: int = 0, hi: int = 12) -> tuple[np.ndarray, np.ndarray]:
    xs = np.empty(n, np.float64)
    ys = np.empty(n, np.float64)
    rc = N.load().gscan_generate_grid(int(n), int(seed), lo, hi, _dptr(xs), _dptr(ys))
    if rc:
        raise ValueError(N.status_string(rc))
    return xs, ys
