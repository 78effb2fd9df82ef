"""TEST INFRASTRUCTURE ONLY — the checker, never the thing measured or shipped.

ctypes front-ends for the two CPU oracles of this repo:
  * ``Ref``: the UNMODIFIED reference library compiled from /root/reference/proj/src by
    oracle/Makefile into oracle/_ref/libcvl_ref.so (entry points in oracle/ref_capi.cpp).
  * ``Restated``: the plain-C restatement oracle/cvl_oracle.c (oracle/_build/libcvl_oracle.so).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
import this module.
"""
from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_LIB = HERE / "_ref" / "libcvl_ref.so"
ORACLE_LIB = HERE / "_build" / "libcvl_oracle.so"

REJECT_NAMES = ["BadTimestamp", "BadNumeric", "MissingField", "RangeViolation", "BadHeader"]
FILTER_NAMES = ["OutOfGrid", "SpeedCeiling", "MissingField"]


class CGrid(ctypes.Structure):
    _fields_ = [("lat_min", ctypes.c_double), ("lat_max", ctypes.c_double),
                ("lon_min", ctypes.c_double), ("lon_max", ctypes.c_double),
                ("lat_step", ctypes.c_double), ("lon_step", ctypes.c_double),
                ("min_step", ctypes.c_uint32), ("dxn_step", ctypes.c_uint32),
                ("dxn_offset", ctypes.c_double)]


class CRules(ctypes.Structure):
    _fields_ = [("require_in_grid", ctypes.c_int32), ("drop_missing", ctypes.c_int32),
                ("speed_ceiling", ctypes.c_double)]


class CStats(ctypes.Structure):
    _fields_ = [("rows_read", ctypes.c_uint64), ("parsed", ctypes.c_uint64),
                ("duplicates_dropped", ctypes.c_uint64),
                ("conflicting_duplicates", ctypes.c_uint64), ("accepted", ctypes.c_uint64),
                ("rejected", ctypes.c_uint64 * 5), ("filtered", ctypes.c_uint64 * 3),
                ("stage_seconds", ctypes.c_double * 4)]

    def as_dict(self) -> dict:
        return {
            "rows_read": self.rows_read, "parsed": self.parsed,
            "duplicates_dropped": self.duplicates_dropped,
            "conflicting_duplicates": self.conflicting_duplicates, "accepted": self.accepted,
            "rejected": {n: int(v) for n, v in zip(REJECT_NAMES, self.rejected) if v},
            "filtered": {n: int(v) for n, v in zip(FILTER_NAMES, self.filtered)},
        }


class CRecordProv(ctypes.Structure):  # ref_record_prov (= cvlg_record in include/cvlg.h)
    _fields_ = [("journey_id", ctypes.c_char_p), ("journey_len", ctypes.c_uint32),
                ("postal_len", ctypes.c_uint32), ("postal_code", ctypes.c_char_p),
                ("shard_path", ctypes.c_char_p), ("shard_path_len", ctypes.c_uint32),
                ("reserved", ctypes.c_uint32), ("line_number", ctypes.c_int64),
                ("epoch_sec", ctypes.c_int64), ("latitude", ctypes.c_double),
                ("longitude", ctypes.c_double), ("speed", ctypes.c_double),
                ("heading", ctypes.c_double)]


def record_array(records):
    """records: (journey_id, epoch_sec, lat, lon, postal, speed, heading, shard_path, line)
    with bytes strings -> ctypes array (the bytes objects stay referenced by the tuples)."""
    arr = (CRecordProv * max(len(records), 1))()
    for i, (jid, ts, la, lo, pc, sp, hd, path, line) in enumerate(records):
        arr[i] = CRecordProv(jid, len(jid), len(pc), pc, path, len(path), 0, line, ts, la, lo, sp, hd)
    return arr


class CRecord(ctypes.Structure):
    _fields_ = [("epoch_sec", ctypes.c_int64), ("latitude", ctypes.c_double),
                ("longitude", ctypes.c_double), ("speed", ctypes.c_double),
                ("heading", ctypes.c_double), ("journey_id", ctypes.c_char * 64),
                ("postal_code", ctypes.c_char * 64)]


def grid_struct(spec) -> CGrid:
    return CGrid(spec.lat_min, spec.lat_max, spec.lon_min, spec.lon_max, spec.lat_step,
                 spec.lon_step, spec.min_step, spec.dxn_step, spec.dxn_offset)


def rules_struct(rules) -> CRules:
    if rules is None:
        return CRules(1, 1, 250.0)
    return CRules(int(rules.require_in_grid), int(rules.drop_missing), rules.speed_ceiling)


def dims(spec) -> tuple[int, int, int, int]:
    """(T, D, R, C) from the reference's own GridSpec math (via ref_bins)."""
    ref = Ref()
    g = grid_struct(spec)
    out = ctypes.c_uint64()
    ref.lib.ref_bins(ctypes.byref(g), 4, 0.0, 0, ctypes.byref(out))
    r = out.value
    ref.lib.ref_bins(ctypes.byref(g), 5, 0.0, 0, ctypes.byref(out))
    c = out.value
    return 1440 // spec.min_step, 360 // spec.dxn_step, r, c


class RefError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        super().__init__(msg)


class Ref:
    """The reference library (oracle/_ref)."""

    _lib = None

    def __init__(self):
        if Ref._lib is None:
            if not REF_LIB.exists():
                raise FileNotFoundError(f"{REF_LIB} not built (make -C oracle ref)")
            lib = ctypes.CDLL(str(REF_LIB))
            vp = ctypes.c_void_p
            lib.ref_run_pipeline.argtypes = [ctypes.POINTER(ctypes.c_char_p), ctypes.c_size_t,
                                             ctypes.POINTER(CGrid), ctypes.POINTER(CRules),
                                             ctypes.c_uint32, ctypes.c_uint32, vp, vp,
                                             ctypes.POINTER(CStats), ctypes.c_char_p,
                                             ctypes.c_size_t]
            lib.ref_run_pipeline_from_records.argtypes = [vp, ctypes.c_size_t,
                                                          ctypes.POINTER(CGrid), ctypes.POINTER(CRules),
                                                          ctypes.c_uint32, ctypes.c_uint32, vp, vp,
                                                          ctypes.POINTER(CStats), ctypes.c_char_p,
                                                          ctypes.c_size_t]
            lib.ref_oracle_pipeline.argtypes = [ctypes.POINTER(ctypes.c_char_p), ctypes.c_size_t,
                                                ctypes.POINTER(CGrid), ctypes.POINTER(CRules),
                                                vp, vp, ctypes.c_char_p, ctypes.c_size_t]
            lib.ref_parse_header.argtypes = [ctypes.c_char_p, ctypes.c_size_t, vp]
            lib.ref_parse_record.argtypes = [ctypes.c_char_p, ctypes.c_size_t, vp,
                                             ctypes.POINTER(CRecord)]
            lib.ref_generate_day.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                             ctypes.c_double, ctypes.c_double, ctypes.c_char_p,
                                             ctypes.c_char_p, vp, ctypes.POINTER(ctypes.c_uint64),
                                             ctypes.c_char_p, ctypes.c_size_t]
            lib.ref_generate_day_mt.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                                ctypes.c_double, ctypes.c_double, ctypes.c_char_p,
                                                ctypes.c_char_p, ctypes.c_uint32,
                                                ctypes.POINTER(ctypes.c_uint64), ctypes.c_char_p,
                                                ctypes.c_size_t]
            lib.ref_write_container.argtypes = [vp, ctypes.POINTER(CGrid), ctypes.c_int32,
                                                ctypes.c_char_p, ctypes.POINTER(ctypes.c_uint64),
                                                ctypes.c_char_p, ctypes.c_size_t]
            lib.ref_bins.argtypes = [ctypes.POINTER(CGrid), ctypes.c_int, ctypes.c_double,
                                     ctypes.c_int64, ctypes.POINTER(ctypes.c_uint64)]
            lib.ref_global_index.argtypes = [ctypes.POINTER(CGrid), ctypes.c_uint32,
                                             ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                             ctypes.POINTER(ctypes.c_uint64)]
            lib.ref_timestamp_parse.argtypes = [ctypes.c_char_p, ctypes.c_size_t,
                                                ctypes.POINTER(ctypes.c_int64)]
            lib.ref_journey_hash.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
            lib.ref_journey_hash.restype = ctypes.c_uint64
            lib.ref_from_chars.argtypes = [ctypes.c_char_p, ctypes.c_size_t,
                                           ctypes.POINTER(ctypes.c_double)]
            lib.ref_deduplicate.argtypes = [ctypes.POINTER(ctypes.c_char_p), ctypes.c_size_t,
                                            vp, vp, vp, ctypes.c_int64,
                                            ctypes.POINTER(ctypes.c_uint64)]
            lib.ref_deduplicate.restype = ctypes.c_int64
            Ref._lib = lib
        self.lib = Ref._lib

    @staticmethod
    def available() -> bool:
        return REF_LIB.exists()

    def run_pipeline(self, paths, spec, rules=None, n_partitions=1, n_threads=1, raw=True):
        """-> (planes [T,8,R,C] u32, raw [T,4,R,C] u32, stats dict)"""
        t, _, r, c = dims(spec)
        planes = np.zeros((t, 8, r, c), dtype=np.uint32)
        rawa = np.zeros((t, 4, r, c), dtype=np.uint32) if raw else None
        arr = (ctypes.c_char_p * max(len(paths), 1))(*[str(p).encode() for p in paths])
        st = CStats()
        err = ctypes.create_string_buffer(512)
        rc = self.lib.ref_run_pipeline(arr, len(paths), ctypes.byref(grid_struct(spec)),
                                       ctypes.byref(rules_struct(rules)), n_partitions, n_threads,
                                       planes.ctypes.data_as(ctypes.c_void_p),
                                       None if rawa is None else rawa.ctypes.data_as(ctypes.c_void_p),
                                       ctypes.byref(st), err, 512)
        if rc:
            raise RefError(rc, err.value.decode())
        return planes, rawa, st.as_dict(), list(st.stage_seconds)

    def run_pipeline_from_records(self, records, spec, rules=None, n_partitions=1, n_threads=1):
        """cvl::run_pipeline_from_records over record tuples (see record_array)"""
        t, _, r, c = dims(spec)
        planes = np.zeros((t, 8, r, c), dtype=np.uint32)
        rawa = np.zeros((t, 4, r, c), dtype=np.uint32)
        arr = record_array(records)
        st = CStats()
        err = ctypes.create_string_buffer(512)
        rc = self.lib.ref_run_pipeline_from_records(ctypes.addressof(arr), len(records),
                                                    ctypes.byref(grid_struct(spec)),
                                                    ctypes.byref(rules_struct(rules)), n_partitions,
                                                    n_threads, planes.ctypes.data_as(ctypes.c_void_p),
                                                    rawa.ctypes.data_as(ctypes.c_void_p),
                                                    ctypes.byref(st), err, 512)
        if rc:
            raise RefError(rc, err.value.decode())
        return planes, rawa, st.as_dict()

    def oracle_pipeline(self, paths, spec, rules=None):
        t, _, r, c = dims(spec)
        planes = np.zeros((t, 8, r, c), dtype=np.uint32)
        rawa = np.zeros((t, 4, r, c), dtype=np.uint32)
        arr = (ctypes.c_char_p * max(len(paths), 1))(*[str(p).encode() for p in paths])
        err = ctypes.create_string_buffer(512)
        rc = self.lib.ref_oracle_pipeline(arr, len(paths), ctypes.byref(grid_struct(spec)),
                                          ctypes.byref(rules_struct(rules)),
                                          planes.ctypes.data_as(ctypes.c_void_p),
                                          rawa.ctypes.data_as(ctypes.c_void_p), err, 512)
        if rc:
            raise RefError(rc, err.value.decode())
        return planes, rawa

    def generate_day(self, out_dir, seed=0, journeys=100, shards=8, sample_period=1.0,
                     mean_duration=300.0, day="2021-05-09", bbox=None) -> int:
        total = ctypes.c_uint64()
        err = ctypes.create_string_buffer(512)
        bb = None
        if bbox is not None:
            bb_arr = (ctypes.c_double * 4)(*bbox)
            bb = ctypes.cast(bb_arr, ctypes.c_void_p)
        rc = self.lib.ref_generate_day(seed, journeys, shards, sample_period, mean_duration,
                                       day.encode(), str(out_dir).encode(), bb,
                                       ctypes.byref(total), err, 512)
        if rc:
            raise RefError(rc, err.value.decode())
        return total.value

    def generate_day_mt(self, out_dir, seed=0, journeys=100, shards=8, sample_period=1.0,
                        mean_duration=300.0, day="2021-05-09", threads=0) -> int:
        """generate_day's files (same bytes), one host thread per shard file."""
        total = ctypes.c_uint64()
        err = ctypes.create_string_buffer(512)
        rc = self.lib.ref_generate_day_mt(seed, journeys, shards, sample_period, mean_duration,
                                          day.encode(), str(out_dir).encode(), threads,
                                          ctypes.byref(total), err, 512)
        if rc:
            raise RefError(rc, err.value.decode())
        return total.value

    def parse_header(self, line: bytes):
        cols = (ctypes.c_int32 * 8)()
        ok = self.lib.ref_parse_header(line, len(line), cols)
        return list(cols) if ok else None

    def parse_record(self, line: bytes, cols):
        carr = (ctypes.c_int32 * 8)(*cols)
        rec = CRecord()
        why = self.lib.ref_parse_record(line, len(line), carr, ctypes.byref(rec))
        return why, rec

    def write_container(self, planes, spec, day, path) -> int:
        n = ctypes.c_uint64()
        err = ctypes.create_string_buffer(512)
        planes = np.ascontiguousarray(planes, dtype=np.uint32)
        rc = self.lib.ref_write_container(planes.ctypes.data_as(ctypes.c_void_p),
                                          ctypes.byref(grid_struct(spec)), day, str(path).encode(),
                                          ctypes.byref(n), err, 512)
        if rc:
            raise RefError(rc, err.value.decode())
        return n.value

    def bin(self, spec, which: int, x: float = 0.0, epoch: int = 0):
        out = ctypes.c_uint64()
        rc = self.lib.ref_bins(ctypes.byref(grid_struct(spec)), which, x, epoch, ctypes.byref(out))
        return (rc, out.value)

    def journey_hash(self, s: bytes) -> int:
        return self.lib.ref_journey_hash(s, len(s))

    def from_chars(self, s: bytes):
        out = ctypes.c_double()
        ok = self.lib.ref_from_chars(s, len(s), ctypes.byref(out))
        return out.value if ok else None

    def timestamp(self, s: bytes):
        out = ctypes.c_int64()
        ok = self.lib.ref_timestamp_parse(s, len(s), ctypes.byref(out))
        return out.value if ok else None


class Restated:
    """The plain-C restatement (oracle/cvl_oracle.c)."""

    _lib = None

    def __init__(self):
        if Restated._lib is None:
            if not ORACLE_LIB.exists():
                raise FileNotFoundError(f"{ORACLE_LIB} not built (make -C oracle oracle)")
            lib = ctypes.CDLL(str(ORACLE_LIB))
            vp = ctypes.c_void_p
            lib.ora_run_pipeline.argtypes = [ctypes.POINTER(ctypes.c_char_p), ctypes.c_size_t,
                                             ctypes.POINTER(CGrid), ctypes.POINTER(CRules), vp, vp,
                                             ctypes.POINTER(CStats), ctypes.c_char_p,
                                             ctypes.c_size_t]
            lib.ora_parse_double.argtypes = [ctypes.c_char_p, ctypes.c_size_t,
                                             ctypes.POINTER(ctypes.c_double)]
            lib.ora_parse_timestamp.argtypes = [ctypes.c_char_p, ctypes.c_size_t,
                                                ctypes.POINTER(ctypes.c_int64)]
            lib.ora_parse_header.argtypes = [ctypes.c_char_p, ctypes.c_size_t, vp]
            lib.ora_parse_record.argtypes = [ctypes.c_char_p, ctypes.c_size_t, vp, vp]
            lib.ora_grid_dims.argtypes = [ctypes.POINTER(CGrid)] + [ctypes.POINTER(ctypes.c_uint32)] * 4
            lib.ora_journey_hash.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
            lib.ora_journey_hash.restype = ctypes.c_uint64
            lib.ora_write_container.argtypes = [vp, ctypes.POINTER(CGrid), ctypes.c_int32,
                                                ctypes.c_char_p, ctypes.POINTER(ctypes.c_uint64)]
            Restated._lib = lib
        self.lib = Restated._lib

    @staticmethod
    def available() -> bool:
        return ORACLE_LIB.exists()

    def dims(self, spec):
        t, d, r, c = (ctypes.c_uint32() for _ in range(4))
        rc = self.lib.ora_grid_dims(ctypes.byref(grid_struct(spec)), ctypes.byref(t), ctypes.byref(d),
                                    ctypes.byref(r), ctypes.byref(c))
        if rc:
            raise RefError(rc, "BadGrid")
        return t.value, d.value, r.value, c.value

    def run_pipeline(self, paths, spec, rules=None, raw=True):
        t, _, r, c = self.dims(spec)
        planes = np.zeros((t, 8, r, c), dtype=np.uint32)
        rawa = np.zeros((t, 4, r, c), dtype=np.uint32) if raw else None
        arr = (ctypes.c_char_p * max(len(paths), 1))(*[str(p).encode() for p in paths])
        st = CStats()
        err = ctypes.create_string_buffer(512)
        rc = self.lib.ora_run_pipeline(arr, len(paths), ctypes.byref(grid_struct(spec)),
                                       ctypes.byref(rules_struct(rules)),
                                       planes.ctypes.data_as(ctypes.c_void_p),
                                       None if rawa is None else rawa.ctypes.data_as(ctypes.c_void_p),
                                       ctypes.byref(st), err, 512)
        if rc:
            raise RefError(rc, err.value.decode())
        return planes, rawa, st.as_dict()

    def parse_double(self, s: bytes):
        out = ctypes.c_double()
        ok = self.lib.ora_parse_double(s, len(s), ctypes.byref(out))
        return out.value if ok else None

    def parse_timestamp(self, s: bytes):
        out = ctypes.c_int64()
        ok = self.lib.ora_parse_timestamp(s, len(s), ctypes.byref(out))
        return out.value if ok else None

    def parse_header(self, line: bytes):
        cols = (ctypes.c_int32 * 8)()
        ok = self.lib.ora_parse_header(line, len(line), cols)
        return list(cols) if ok else None

    def journey_hash(self, s: bytes) -> int:
        return self.lib.ora_journey_hash(s, len(s))
