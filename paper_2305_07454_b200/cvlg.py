"""Python host mirror of the reference pipeline API over the sm_100a C ABI (include/cvlg.h).

Mirrors the reference's public surface for this path:
  * ``run_pipeline(manifest, spec, rules, n_partitions, n_threads, stats)``
    -> cvl::run_pipeline (proj/include/cvl/aggregate.hpp:125-127)
  * ``GridSpec`` / ``FilterRules`` / ``PipelineStats`` / ``BatchFrame``
    -> grid.hpp:21-41, aggregate.hpp:16-20, 112-121, 46-57
  * ``write_container`` -> lattice_store.hpp:43-44 (.cvl1 bytes)
  * ``CvlError`` with the reference's Err codes (error.hpp:8-26)

There is no CPU fallback: importing this module fails loudly when the CUDA library is missing,
and every compute call runs the sm_100a kernels.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from pathlib import Path
from typing import Iterable, Sequence

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "lib" / "libcvlg.so"
if os.environ.get("CVLG_LIB_VARIANT"):  # A/B builds of the same sources (tools/, never the default)
    LIB_PATH = _HERE / "lib" / f"libcvlg.{os.environ['CVLG_LIB_VARIANT']}.so"

ERR_NAMES = [
    "MissingRoot", "BadConfig", "BadGrid", "ZeroPartitions", "OutOfBounds",
    "ComponentOutOfRange", "IndexOverflow", "GridMismatch", "DimsMismatch", "NonFiniteValue",
    "Io", "BadMagic", "VersionUnsupported", "TruncatedFile", "BadChannel", "TaskFailed",
    "DivideByZero",
]
EXTRA_ERRS = {100: "Cuda", 101: "InvalidArgument", 102: "Unsupported", 103: "Internal"}
REJECT_NAMES = ["BadTimestamp", "BadNumeric", "MissingField", "RangeViolation", "BadHeader"]
FILTER_NAMES = ["OutOfGrid", "SpeedCeiling", "MissingField"]
STAGE_NAMES = ["parse", "dedup+filter+accumulate", "merge", "finalize"]  # aggregate.cpp:370-383, 449


class CvlError(RuntimeError):
    """Mirror of cvl::CvlError: ``code`` is the reference Err name (or a CVLG extra)."""

    def __init__(self, status: int, message: str):
        if 1 <= status <= len(ERR_NAMES):
            self.code = ERR_NAMES[status - 1]
        else:
            self.code = EXTRA_ERRS.get(status, f"Status{status}")
        self.status = status
        super().__init__(message or self.code)


class _Grid(ctypes.Structure):
    _fields_ = [("lat_min", ctypes.c_double), ("lat_max", ctypes.c_double),
                ("lon_min", ctypes.c_double), ("lon_max", ctypes.c_double),
                ("lat_step", ctypes.c_double), ("lon_step", ctypes.c_double),
                ("min_step", ctypes.c_uint32), ("dxn_step", ctypes.c_uint32),
                ("dxn_offset", ctypes.c_double)]


class _Rules(ctypes.Structure):
    _fields_ = [("require_in_grid", ctypes.c_int32), ("drop_missing", ctypes.c_int32),
                ("speed_ceiling", ctypes.c_double)]


class _Stats(ctypes.Structure):
    _fields_ = [("rows_read", ctypes.c_uint64), ("parsed", ctypes.c_uint64),
                ("duplicates_dropped", ctypes.c_uint64),
                ("conflicting_duplicates", ctypes.c_uint64), ("accepted", ctypes.c_uint64),
                ("rejected", ctypes.c_uint64 * 5), ("filtered", ctypes.c_uint64 * 3),
                ("stage_seconds", ctypes.c_double * 4)]


class _Features(ctypes.Structure):
    _fields_ = [("n_journeys", ctypes.c_uint64)] + [
        (n, ctypes.c_void_p) for n in ("points", "t_first", "t_last", "length_m", "max_step_m",
                                       "max_speed", "max_abs_accel", "dwell_s", "stops", "id_span",
                                       "cell_speed_min", "cell_speed_max")]


def _load() -> ctypes.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: the sm_100a library is not built "
            "(run `python -c 'import __graft_entry__ as g; g.build()'`). There is no CPU fallback.")
    lib = ctypes.CDLL(str(LIB_PATH))
    u32p = ctypes.POINTER(ctypes.c_uint32)
    u64p = ctypes.POINTER(ctypes.c_uint64)
    vp = ctypes.c_void_p
    lib.cvlg_context_create.restype = vp
    lib.cvlg_context_create.argtypes = [ctypes.c_int]
    lib.cvlg_context_destroy.argtypes = [vp]
    lib.cvlg_grid_dims.argtypes = [ctypes.POINTER(_Grid), u32p, u32p, u32p, u32p]
    lib.cvlg_run_pipeline.argtypes = [vp, ctypes.POINTER(ctypes.c_char_p), ctypes.c_size_t,
                                      ctypes.POINTER(_Grid), ctypes.POINTER(_Rules),
                                      ctypes.c_uint32, ctypes.c_uint32, vp, vp,
                                      ctypes.POINTER(_Stats)]
    lib.cvlg_run_pipeline_host.argtypes = [vp, ctypes.POINTER(vp), u64p, ctypes.c_size_t,
                                           ctypes.POINTER(_Grid), ctypes.POINTER(_Rules),
                                           ctypes.c_uint32, vp, vp, ctypes.POINTER(_Stats)]
    lib.cvlg_run_pipeline_records.argtypes = [vp, vp, ctypes.c_size_t, ctypes.POINTER(_Grid),
                                              ctypes.POINTER(_Rules), ctypes.c_uint32,
                                              ctypes.c_uint32, vp, vp, ctypes.POINTER(_Stats)]
    lib.cvlg_run_pipeline_device.argtypes = [vp, vp, u64p, ctypes.c_size_t,
                                             ctypes.POINTER(_Grid), ctypes.POINTER(_Rules), vp,
                                             vp, ctypes.POINTER(_Stats), vp]
    lib.cvlg_write_container.argtypes = [vp, ctypes.POINTER(_Grid), ctypes.c_int32,
                                         ctypes.c_char_p, u64p]
    lib.cvlg_last_stage_ms.argtypes = [vp, ctypes.POINTER(ctypes.c_float), ctypes.c_int]
    lib.cvlg_context_input.argtypes = [vp, ctypes.POINTER(vp), u64p]
    lib.cvlg_pin_host.argtypes = [vp, ctypes.c_size_t]
    lib.cvlg_unpin_host.argtypes = [vp]
    lib.cvlg_launch_count.restype = ctypes.c_uint64
    lib.cvlg_last_error.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
    lib.cvlg_journey_features_host.argtypes = [vp, ctypes.POINTER(vp), u64p, ctypes.c_size_t,
                                               ctypes.POINTER(_Grid), ctypes.POINTER(_Rules),
                                               ctypes.c_double, vp, vp, ctypes.POINTER(_Stats),
                                               u64p]
    lib.cvlg_journey_features_device.argtypes = [vp, vp, u64p, ctypes.c_size_t,
                                                 ctypes.POINTER(_Grid), ctypes.POINTER(_Rules),
                                                 ctypes.c_double, vp, vp, ctypes.POINTER(_Stats),
                                                 u64p, vp]
    lib.cvlg_features_copy.argtypes = [vp, ctypes.POINTER(_Features)]
    # multi-GPU (include/cvlg.h, multi.cu)
    lib.cvlg_multi_create.restype = vp
    lib.cvlg_multi_create.argtypes = [ctypes.POINTER(ctypes.c_int), ctypes.c_uint32]
    lib.cvlg_multi_destroy.argtypes = [vp]
    lib.cvlg_multi_size.restype = ctypes.c_uint32
    lib.cvlg_multi_size.argtypes = [vp]
    lib.cvlg_multi_context.restype = vp
    lib.cvlg_multi_context.argtypes = [vp, ctypes.c_uint32]
    lib.cvlg_run_pipeline_multi.argtypes = [vp, ctypes.POINTER(ctypes.c_char_p), ctypes.c_size_t,
                                            ctypes.POINTER(_Grid), ctypes.POINTER(_Rules),
                                            ctypes.c_uint32, ctypes.c_uint32, vp, vp,
                                            ctypes.POINTER(_Stats)]
    lib.cvlg_route_stage.argtypes = [vp, ctypes.POINTER(ctypes.c_char_p), ctypes.c_size_t,
                                     ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, u64p, u64p]
    lib.cvlg_route_count.argtypes = [vp]
    lib.cvlg_route_plan.argtypes = [vp, ctypes.c_uint32, u64p, u64p]
    lib.cvlg_route_scatter.argtypes = [vp, ctypes.POINTER(vp), vp]
    lib.cvlg_tuples_export.argtypes = [vp, ctypes.POINTER(_Grid), ctypes.c_uint32, vp, u64p, u64p]
    lib.cvlg_partial_info.argtypes = [vp, u64p, u64p, ctypes.POINTER(ctypes.c_int32)]
    lib.cvlg_journey_ids.argtypes = [vp, vp, ctypes.c_uint64, u64p, ctypes.c_uint64, u64p, u64p]
    lib.cvlg_merge_id_ranks.argtypes = [ctypes.c_uint32, ctypes.POINTER(vp), ctypes.POINTER(vp),
                                        u64p, ctypes.POINTER(vp)]
    lib.cvlg_tuples_scatter.argtypes = [vp, ctypes.POINTER(_Grid), ctypes.c_uint32,
                                        ctypes.POINTER(vp), vp]
    lib.cvlg_finalize_tuples.argtypes = [vp, vp, ctypes.c_uint64, ctypes.POINTER(_Grid),
                                         ctypes.c_uint32, ctypes.c_uint32, vp, vp, vp]
    lib.cvlg_slab_rows.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, u32p, u32p]
    lib.cvlg_split_manifest.argtypes = [ctypes.POINTER(ctypes.c_char_p), ctypes.c_size_t,
                                        ctypes.c_uint32, ctypes.c_uint32, u32p, u64p, u64p,
                                        ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
    lib.cvlg_partial_device.argtypes = [vp, vp, u64p, ctypes.c_size_t, ctypes.POINTER(_Grid),
                                        ctypes.POINTER(_Rules), u64p, ctypes.POINTER(_Stats), vp]
    lib.cvlg_export_pairs.argtypes = [vp, vp, vp, vp, vp, vp, vp]
    lib.cvlg_finalize_pairs.argtypes = [vp, vp, vp, vp, vp, vp, ctypes.c_uint64,
                                        ctypes.POINTER(_Grid), vp, vp, vp]
    return lib


_lib = _load()

EXPORTED_SYMBOLS = [
    "cvlg_default_grid", "cvlg_default_rules", "cvlg_grid_dims", "cvlg_context_create",
    "cvlg_context_destroy", "cvlg_run_pipeline", "cvlg_run_pipeline_host",
    "cvlg_run_pipeline_device", "cvlg_write_container", "cvlg_last_stage_ms", "cvlg_pin_host",
    "cvlg_unpin_host", "cvlg_launch_count", "cvlg_last_error", "cvlg_journey_features_host",
    "cvlg_journey_features_device", "cvlg_features_copy", "cvlg_context_input",
    "cvlg_multi_create", "cvlg_multi_destroy", "cvlg_multi_size", "cvlg_multi_context",
    "cvlg_run_pipeline_multi", "cvlg_route_stage", "cvlg_route_count", "cvlg_route_plan",
    "cvlg_route_scatter", "cvlg_tuples_export", "cvlg_tuples_scatter", "cvlg_finalize_tuples",
    "cvlg_slab_rows", "cvlg_split_manifest", "cvlg_partial_device", "cvlg_partial_info",
    "cvlg_journey_ids", "cvlg_merge_id_ranks", "cvlg_export_pairs", "cvlg_finalize_pairs",
]


def lib() -> ctypes.CDLL:
    return _lib


def _check(status: int) -> None:
    if status != 0:
        buf = ctypes.create_string_buffer(1024)
        _lib.cvlg_last_error(buf, 1024)
        raise CvlError(status, buf.value.decode(errors="replace"))


@dataclass
class GridSpec:
    """cvl::GridSpec (grid.hpp:21-41), same defaults."""

    lat_min: float = 36.0
    lat_max: float = 40.6
    lon_min: float = -95.8
    lon_max: float = -89.1
    lat_step: float = 0.1
    lon_step: float = 0.1
    min_step: int = 5
    dxn_step: int = 90
    dxn_offset: float = 0.0

    def _c(self) -> _Grid:
        return _Grid(self.lat_min, self.lat_max, self.lon_min, self.lon_max, self.lat_step,
                     self.lon_step, self.min_step, self.dxn_step, self.dxn_offset)

    def dims(self) -> tuple[int, int, int, int]:
        """(T, D, R, C); raises CvlError(BadGrid) like GridSpec::validate."""
        t, d, r, c = (ctypes.c_uint32() for _ in range(4))
        _check(_lib.cvlg_grid_dims(ctypes.byref(self._c()), ctypes.byref(t), ctypes.byref(d),
                                   ctypes.byref(r), ctypes.byref(c)))
        return t.value, d.value, r.value, c.value

    def validate(self) -> None:
        self.dims()

    @property
    def rows(self) -> int:
        return self.dims()[2]

    @property
    def cols(self) -> int:
        return self.dims()[3]

    def batches(self) -> int:
        return 1440 // self.min_step

    def directions(self) -> int:
        return 360 // self.dxn_step

    def cell_count(self) -> int:
        t, d, r, c = self.dims()
        return t * d * r * c


@dataclass
class FilterRules:
    """cvl::FilterRules (aggregate.hpp:16-20)."""

    require_in_grid: bool = True
    speed_ceiling: float = 250.0
    drop_missing: bool = True

    def _c(self) -> _Rules:
        return _Rules(int(self.require_in_grid), int(self.drop_missing), self.speed_ceiling)


@dataclass
class PipelineStats:
    """cvl::PipelineStats (aggregate.hpp:112-121)."""

    rows_read: int = 0
    parsed: int = 0
    duplicates_dropped: int = 0
    conflicting_duplicates: int = 0
    accepted: int = 0
    rejected: dict = field(default_factory=dict)
    filtered: dict = field(default_factory=dict)
    stage_seconds: list = field(default_factory=list)

    def _fill(self, s: _Stats) -> None:
        self.rows_read = s.rows_read
        self.parsed = s.parsed
        self.duplicates_dropped = s.duplicates_dropped
        self.conflicting_duplicates = s.conflicting_duplicates
        self.accepted = s.accepted
        # the reference's rejected map only holds reasons that occurred (aggregate.cpp:446-447)
        self.rejected = {n: int(v) for n, v in zip(REJECT_NAMES, s.rejected) if v}
        self.filtered = {n: int(v) for n, v in zip(FILTER_NAMES, s.filtered)}
        self.stage_seconds = [(n, float(v)) for n, v in zip(STAGE_NAMES, s.stage_seconds)]


class BatchFrame:
    """cvl::BatchFrame view (aggregate.hpp:46-57) over one t-slab of a Lattice."""

    def __init__(self, t: int, planes: np.ndarray, raw: np.ndarray | None):
        self.t = t
        self.rows, self.cols = planes.shape[-2], planes.shape[-1]
        self.speed = [planes[d].view(np.float32) for d in range(4)]
        self.volume = [planes[4 + d] for d in range(4)]
        self.raw_count = [raw[d] for d in range(4)] if raw is not None else None

    def bitwise_equal(self, other: "BatchFrame") -> bool:
        """t, dims, speed bit patterns and volumes; raw_count excluded (aggregate.cpp:145-159)."""
        if (self.t, self.rows, self.cols) != (other.t, other.rows, other.cols):
            return False
        return all(np.array_equal(self.speed[d].view(np.uint32), other.speed[d].view(np.uint32))
                   and np.array_equal(self.volume[d], other.volume[d]) for d in range(4))


class Lattice(Sequence):
    """The T BatchFrames of one run, stored densely: planes [T][8][R][C] u32 (speed f32 bits
    for d = 0..3, then volume) and raw_count [T][4][R][C] u32."""

    def __init__(self, planes: np.ndarray, raw: np.ndarray | None):
        self.planes = planes
        self.raw = raw

    def __len__(self) -> int:
        return self.planes.shape[0]

    def __getitem__(self, t):
        if isinstance(t, slice):
            return [self[i] for i in range(*t.indices(len(self)))]
        return BatchFrame(t, self.planes[t], None if self.raw is None else self.raw[t])

    @property
    def speed(self) -> np.ndarray:
        return self.planes[:, :4].view(np.float32)

    @property
    def volume(self) -> np.ndarray:
        return self.planes[:, 4:]


def _alloc(spec: GridSpec, raw: bool):
    t, _, r, c = spec.dims()
    planes = np.empty((t, 8, r, c), dtype=np.uint32)
    rawa = np.empty((t, 4, r, c), dtype=np.uint32) if raw else None
    return planes, rawa


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class Context:
    """Owns a device context (streams + grow-only scratch). One per host thread."""

    def __init__(self, device: int = -1):
        self._h = _lib.cvlg_context_create(device)
        if not self._h:
            buf = ctypes.create_string_buffer(1024)
            _lib.cvlg_last_error(buf, 1024)
            raise CvlError(100, buf.value.decode() or "cvlg_context_create failed")

    @property
    def handle(self):
        return self._h

    def close(self) -> None:
        if self._h:
            _lib.cvlg_context_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def input(self) -> tuple[int, int]:
        """(device pointer, bytes) of the input the last file/host run left resident in HBM."""
        p = ctypes.c_void_p()
        n = ctypes.c_uint64()
        _check(_lib.cvlg_context_input(self._h, ctypes.byref(p), ctypes.byref(n)))
        return int(p.value or 0), int(n.value)

    def stage_ms(self) -> list[float]:
        """[parse, dedup+filter+accumulate, merge, finalize, decode kernel, dictionary+order]"""
        arr = (ctypes.c_float * 6)()
        _lib.cvlg_last_stage_ms(self._h, arr, 6)
        return list(arr)


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context()
    return _default_ctx


def _paths(manifest) -> list[str]:
    if hasattr(manifest, "shard_paths"):
        return [str(p) for p in manifest.shard_paths]
    return [str(p) for p in manifest]


def run_pipeline(manifest, spec: GridSpec | None = None, rules: FilterRules | None = None,
                 n_partitions: int = 1, n_threads: int = 0,
                 stats: PipelineStats | None = None, ctx: Context | None = None,
                 raw: bool = True, out: tuple | None = None) -> Lattice:
    """cvl::run_pipeline (aggregate.hpp:125-127): shard files -> lattice, on the GPU. The files
    stream through a bounded pinned ring (n_threads reader threads) into HBM while decode runs.
    `out` = (planes, raw) host arrays to fill (e.g. pinned) instead of fresh ones."""
    spec = spec or GridSpec()
    rules = rules or FilterRules()
    ctx = ctx or default_context()
    paths = _paths(manifest)
    arr = (ctypes.c_char_p * max(len(paths), 1))(*[p.encode() for p in paths])
    planes, rawa = out if out is not None else _alloc(spec, raw)
    st = _Stats()
    _check(_lib.cvlg_run_pipeline(ctx.handle, arr, len(paths), ctypes.byref(spec._c()),
                                  ctypes.byref(rules._c()), n_partitions, n_threads,
                                  _ptr(planes), _ptr(rawa), ctypes.byref(st)))
    if stats is not None:
        stats._fill(st)
    return Lattice(planes, rawa)


class MultiGPU:
    """Several GPUs driven from one host thread (cvlg_multi_*): journeys sharded by
    journey_hash(id) % n like the reference's partitions (aggregate.cpp:414-443). `devices` may
    repeat a device (several shards on one GPU)."""

    def __init__(self, devices: Sequence[int]):
        arr = (ctypes.c_int * len(devices))(*devices)
        self._h = _lib.cvlg_multi_create(arr, len(devices))
        if not self._h:
            buf = ctypes.create_string_buffer(1024)
            _lib.cvlg_last_error(buf, 1024)
            raise CvlError(100, buf.value.decode() or "cvlg_multi_create failed")
        self.devices = list(devices)

    @property
    def handle(self):
        return self._h

    def __len__(self) -> int:
        return len(self.devices)

    def close(self) -> None:
        if self._h:
            _lib.cvlg_multi_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run_pipeline(self, manifest, spec: GridSpec | None = None, rules: FilterRules | None = None,
                     n_partitions: int = 1, n_threads: int = 0, stats: PipelineStats | None = None,
                     raw: bool = True, out: tuple | None = None) -> Lattice:
        """cvl::run_pipeline over the group's GPUs (cvlg_run_pipeline_multi): same result as
        run_pipeline on one GPU, byte for byte."""
        spec = spec or GridSpec()
        rules = rules or FilterRules()
        paths = _paths(manifest)
        arr = (ctypes.c_char_p * max(len(paths), 1))(*[p.encode() for p in paths])
        planes, rawa = out if out is not None else _alloc(spec, raw)
        st = _Stats()
        _check(_lib.cvlg_run_pipeline_multi(self._h, arr, len(paths), ctypes.byref(spec._c()),
                                            ctypes.byref(rules._c()), n_partitions, n_threads,
                                            _ptr(planes), _ptr(rawa), ctypes.byref(st)))
        if stats is not None:
            stats._fill(st)
        return Lattice(planes, rawa)


def split_manifest(manifest, n_parts: int, part: int) -> list[tuple[int, int, int]]:
    """Host only: the (file rank, byte offset, length) pieces of part `part` of `n_parts` as the
    multi-GPU ingest cuts the shards' data lines (cvlg_split_manifest)."""
    paths = _paths(manifest)
    arr = (ctypes.c_char_p * max(len(paths), 1))(*[p.encode() for p in paths])
    n = ctypes.c_size_t()
    _check(_lib.cvlg_split_manifest(arr, len(paths), n_parts, part, None, None, None, 0,
                                    ctypes.byref(n)))
    k = n.value
    f = (ctypes.c_uint32 * max(k, 1))()
    o = (ctypes.c_uint64 * max(k, 1))()
    ln = (ctypes.c_uint64 * max(k, 1))()
    _check(_lib.cvlg_split_manifest(arr, len(paths), n_parts, part, f, o, ln, k, ctypes.byref(n)))
    return [(int(f[i]), int(o[i]), int(ln[i])) for i in range(k)]


def slab_rows(n_batches: int, n_owners: int, owner: int) -> tuple[int, int]:
    """Rows [t0, t1) of the lattice folded by slab owner `owner` (cvlg_slab_rows)."""
    t0, t1 = ctypes.c_uint32(), ctypes.c_uint32()
    _check(_lib.cvlg_slab_rows(n_batches, n_owners, owner, ctypes.byref(t0), ctypes.byref(t1)))
    return t0.value, t1.value


def run_pipeline_host(buffers: Iterable, spec: GridSpec | None = None,
                      rules: FilterRules | None = None, n_partitions: int = 1,
                      stats: PipelineStats | None = None, ctx: Context | None = None,
                      raw: bool = True, out: tuple | None = None) -> Lattice:
    """Shard bytes in host memory (rank order) -> lattice. Buffers: bytes / uint8 ndarrays."""
    spec = spec or GridSpec()
    rules = rules or FilterRules()
    ctx = ctx or default_context()
    keep = []
    ptrs, lens = [], []
    for b in buffers:
        a = np.frombuffer(b, dtype=np.uint8) if isinstance(b, (bytes, bytearray, memoryview)) else b
        keep.append(a)
        ptrs.append(a.ctypes.data if a.size else 0)
        lens.append(a.size)
    n = len(ptrs)
    parr = (ctypes.c_void_p * max(n, 1))(*ptrs)
    larr = (ctypes.c_uint64 * max(n, 1))(*lens)
    planes, rawa = out if out is not None else _alloc(spec, raw)
    st = _Stats()
    _check(_lib.cvlg_run_pipeline_host(ctx.handle, parr, larr, n, ctypes.byref(spec._c()),
                                       ctypes.byref(rules._c()), n_partitions, _ptr(planes),
                                       _ptr(rawa), ctypes.byref(st)))
    if stats is not None:
        stats._fill(st)
    return Lattice(planes, rawa)


class _Record(ctypes.Structure):  # cvlg_record (include/cvlg.h)
    _fields_ = [("journey_id", ctypes.c_char_p), ("journey_len", ctypes.c_uint32),
                ("postal_len", ctypes.c_uint32), ("postal_code", ctypes.c_char_p),
                ("shard_path", ctypes.c_char_p), ("shard_path_len", ctypes.c_uint32),
                ("reserved", ctypes.c_uint32), ("line_number", ctypes.c_int64),
                ("epoch_sec", ctypes.c_int64), ("latitude", ctypes.c_double),
                ("longitude", ctypes.c_double), ("speed", ctypes.c_double),
                ("heading", ctypes.c_double)]


def run_pipeline_from_records(records: Sequence, spec: GridSpec | None = None,
                              rules: FilterRules | None = None, n_partitions: int = 1,
                              n_threads: int = 0, stats: PipelineStats | None = None,
                              ctx: Context | None = None, raw: bool = True) -> Lattice:
    """cvl::run_pipeline_from_records (aggregate.hpp:130-133): already-parsed records with
    provenance -> lattice. Each record is (journey_id, epoch_sec, latitude, longitude,
    postal_code, speed, heading, shard_path, line_number); strings as bytes."""
    spec = spec or GridSpec()
    rules = rules or FilterRules()
    ctx = ctx or default_context()
    arr = (_Record * max(len(records), 1))()
    for i, (jid, ts, la, lo, pc, sp, hd, path, line) in enumerate(records):
        arr[i] = _Record(jid, len(jid), len(pc), pc, path, len(path), 0, line, ts, la, lo, sp, hd)
    planes, rawa = _alloc(spec, raw)
    st = _Stats()
    _check(_lib.cvlg_run_pipeline_records(ctx.handle, ctypes.addressof(arr), len(records),
                                          ctypes.byref(spec._c()), ctypes.byref(rules._c()),
                                          n_partitions, n_threads, _ptr(planes), _ptr(rawa),
                                          ctypes.byref(st)))
    if stats is not None:
        stats._fill(st)
    return Lattice(planes, rawa)


def run_pipeline_device(d_csv_ptr: int, shard_offsets: Sequence[int], d_planes_ptr: int,
                        d_raw_ptr: int | None = None, spec: GridSpec | None = None,
                        rules: FilterRules | None = None, stats: PipelineStats | None = None,
                        ctx: Context | None = None, stream: int | None = None) -> None:
    """Device-resident pipeline: CSV bytes and output lattice in HBM (raw device pointers,
    e.g. ``tensor.data_ptr()``)."""
    spec = spec or GridSpec()
    rules = rules or FilterRules()
    ctx = ctx or default_context()
    offs = (ctypes.c_uint64 * len(shard_offsets))(*shard_offsets)
    st = _Stats()
    _check(_lib.cvlg_run_pipeline_device(ctx.handle, ctypes.c_void_p(d_csv_ptr), offs,
                                         len(shard_offsets) - 1, ctypes.byref(spec._c()),
                                         ctypes.byref(rules._c()), ctypes.c_void_p(d_planes_ptr),
                                         ctypes.c_void_p(d_raw_ptr) if d_raw_ptr else None,
                                         ctypes.byref(st),
                                         ctypes.c_void_p(stream) if stream else None))
    if stats is not None:
        stats._fill(st)


FEATURE_COLUMNS = {
    "points": np.uint32, "t_first": np.int64, "t_last": np.int64, "length_m": np.float64,
    "max_step_m": np.float64, "max_speed": np.float64, "max_abs_accel": np.float64,
    "dwell_s": np.float64, "stops": np.uint32, "id_span": np.uint64,
}


def _features_fetch(ctx: Context, spec: GridSpec, n: int) -> dict:
    out = {k: np.empty(n, dtype=t) for k, t in FEATURE_COLUMNS.items()}
    t, _, r, c = spec.dims()
    out["cell_speed_min"] = np.empty((t, 4, r, c), dtype=np.float32)
    out["cell_speed_max"] = np.empty((t, 4, r, c), dtype=np.float32)
    f = _Features()
    for k, a in out.items():
        setattr(f, k, a.ctypes.data if a.size else None)
    _check(_lib.cvlg_features_copy(ctx.handle, ctypes.byref(f)))
    return out


def journey_features_host(buffers: Iterable, spec: GridSpec | None = None,
                          rules: FilterRules | None = None, stop_speed: float = 5.0,
                          stats: PipelineStats | None = None, ctx: Context | None = None):
    """Pipeline + per-journey feature table (north_star extension, NOT in the reference; see
    include/cvlg.h cvlg_journey_features_host). Returns (Lattice, features dict): one row per
    journey in lexicographic id order; ``id_span`` = byte offset | length << 40 into the
    concatenated shard bytes; ``journey_ids(buffers, features)`` decodes them."""
    spec = spec or GridSpec()
    rules = rules or FilterRules()
    ctx = ctx or default_context()
    keep, ptrs, lens = [], [], []
    for b in buffers:
        a = np.frombuffer(b, dtype=np.uint8) if isinstance(b, (bytes, bytearray, memoryview)) else b
        keep.append(a)
        ptrs.append(a.ctypes.data if a.size else 0)
        lens.append(a.size)
    n = len(ptrs)
    parr = (ctypes.c_void_p * max(n, 1))(*ptrs)
    larr = (ctypes.c_uint64 * max(n, 1))(*lens)
    planes, rawa = _alloc(spec, True)
    st = _Stats()
    nj = ctypes.c_uint64()
    _check(_lib.cvlg_journey_features_host(ctx.handle, parr, larr, n, ctypes.byref(spec._c()),
                                           ctypes.byref(rules._c()), float(stop_speed),
                                           _ptr(planes), _ptr(rawa), ctypes.byref(st),
                                           ctypes.byref(nj)))
    if stats is not None:
        stats._fill(st)
    return Lattice(planes, rawa), _features_fetch(ctx, spec, nj.value)


def journey_features_device(d_csv_ptr: int, shard_offsets: Sequence[int], d_planes_ptr: int,
                            d_raw_ptr: int | None = None, spec: GridSpec | None = None,
                            rules: FilterRules | None = None, stop_speed: float = 5.0,
                            stats: PipelineStats | None = None, ctx: Context | None = None,
                            stream: int | None = None, fetch: bool = True):
    """Device-resident pipeline + per-journey features (see journey_features_host). Returns the
    features dict (host copies) when ``fetch``, else the number of journeys."""
    spec = spec or GridSpec()
    rules = rules or FilterRules()
    ctx = ctx or default_context()
    offs = (ctypes.c_uint64 * len(shard_offsets))(*shard_offsets)
    st = _Stats()
    nj = ctypes.c_uint64()
    _check(_lib.cvlg_journey_features_device(
        ctx.handle, ctypes.c_void_p(d_csv_ptr), offs, len(shard_offsets) - 1,
        ctypes.byref(spec._c()), ctypes.byref(rules._c()), float(stop_speed),
        ctypes.c_void_p(d_planes_ptr), ctypes.c_void_p(d_raw_ptr) if d_raw_ptr else None,
        ctypes.byref(st), ctypes.byref(nj), ctypes.c_void_p(stream) if stream else None))
    if stats is not None:
        stats._fill(st)
    return _features_fetch(ctx, spec, nj.value) if fetch else nj.value


def journey_ids(buffers: Iterable, features: dict) -> list[bytes]:
    """Journey id bytes of each feature row (id_span into the concatenated shard bytes)."""
    blob = b"".join(bytes(b) for b in buffers)
    spans = features["id_span"]
    return [blob[int(s) & ((1 << 40) - 1):(int(s) & ((1 << 40) - 1)) + (int(s) >> 40)] for s in spans]


def write_container(frames: Lattice | np.ndarray, spec: GridSpec, day: int, path: str | os.PathLike) -> int:
    """cvl::write_container (lattice_store.cpp:78-134): returns bytes written."""
    planes = frames.planes if isinstance(frames, Lattice) else frames
    planes = np.ascontiguousarray(planes, dtype=np.uint32)
    n = ctypes.c_uint64()
    _check(_lib.cvlg_write_container(_ptr(planes), ctypes.byref(spec._c()), day,
                                     str(path).encode(), ctypes.byref(n)))
    return n.value


def pin_host(a: np.ndarray) -> None:
    _check(_lib.cvlg_pin_host(a.ctypes.data, a.nbytes))


def unpin_host(a: np.ndarray) -> None:
    _check(_lib.cvlg_unpin_host(a.ctypes.data))


def launch_count() -> int:
    return int(_lib.cvlg_launch_count())


def synth_day(seed: int = 0, journeys: int = 100, shards: int = 8, sample_period: float = 1.0,
              mean_duration: float = 300.0, day: str = "2021-05-09", bbox=None,
              threads: int = 0):
    """Threaded in-memory twin of the reference generate_day (synth.cpp:145-181), byte-identical
    output. Returns (blob uint8 ndarray, shard offsets list[int], total_rows)."""
    import datetime
    d = datetime.date.fromisoformat(day)
    day_number = (d - datetime.date(1970, 1, 1)).days
    max_rows = journeys * (int(1.7 * mean_duration / sample_period) + 2)
    cap = max_rows * 80 + shards * 80 + 64
    out = np.empty(cap, dtype=np.uint8)
    offs = (ctypes.c_uint64 * (shards + 1))()
    rows = ctypes.c_uint64()
    bb = (ctypes.c_double * 4)(*bbox) if bbox is not None else None
    fn = _lib.cvlg_synth_day
    fn.restype = ctypes.c_int64
    fn.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_double,
                   ctypes.c_double, ctypes.c_int32, ctypes.c_void_p, ctypes.c_uint32,
                   ctypes.c_void_p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64),
                   ctypes.POINTER(ctypes.c_uint64)]
    n = fn(seed, journeys, shards, sample_period, mean_duration, day_number,
           ctypes.cast(bb, ctypes.c_void_p) if bb is not None else None, threads,
           out.ctypes.data_as(ctypes.c_void_p), cap, offs, ctypes.byref(rows))
    if n < 0:
        raise CvlError(101, f"synth_day failed ({n})")
    return out[:n], list(offs), rows.value


def synth_write_day(out_dir, seed: int = 0, journeys: int = 100, shards: int = 8,
                    sample_period: float = 1.0, mean_duration: float = 300.0,
                    day: str = "2021-05-09", threads: int = 0) -> tuple[int, int]:
    """Writes the reference generate_day's shard files (byte-identical, synth.cpp:145-181) to
    out_dir with one host thread per file. Returns (bytes, rows)."""
    import datetime
    d = datetime.date.fromisoformat(day)
    day_number = (d - datetime.date(1970, 1, 1)).days
    os.makedirs(out_dir, exist_ok=True)
    rows = ctypes.c_uint64()
    fn = _lib.cvlg_synth_write_day
    fn.restype = ctypes.c_int64
    fn.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_double,
                   ctypes.c_double, ctypes.c_int32, ctypes.c_uint32, ctypes.c_char_p,
                   ctypes.POINTER(ctypes.c_uint64)]
    n = fn(seed, journeys, shards, sample_period, mean_duration, day_number, threads,
           str(out_dir).encode(), ctypes.byref(rows))
    if n < 0:
        raise CvlError(11 if n == -3 else 101, f"synth_write_day failed ({n})")
    return int(n), rows.value


def shuffle_rows(blob: np.ndarray, offs: Sequence[int], n_out: int, seed: int = 7,
                 header: bytes = b"Journey Id,Timestamp,Latitude,Longitude,Postal Code,Speed,Heading"):
    """Adversarial variant: all data rows shuffled across n_out shards (C++)."""
    out = np.empty(int(offs[-1]) + n_out * (len(header) + 1) + 64, dtype=np.uint8)
    ooffs = (ctypes.c_uint64 * (n_out + 1))()
    iof = (ctypes.c_uint64 * len(offs))(*offs)
    fn = _lib.cvlg_shuffle_rows
    fn.restype = ctypes.c_int64
    fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_char_p,
                   ctypes.c_uint32, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]
    n = fn(blob.ctypes.data_as(ctypes.c_void_p), iof, len(offs) - 1, seed, header, n_out,
           out.ctypes.data_as(ctypes.c_void_p), out.size, ooffs)
    if n < 0:
        raise CvlError(101, f"shuffle_rows failed ({n})")
    return out[:n], list(ooffs)
