"""CPU tests (no GPU): the product's device decode logic (csrc/parse.cuh + grid.cuh) compiled for
the host (tests/native/hostparse.cpp) against the golden vectors from the reference. The same
source is compiled for sm_100a; tests/test_gpu_parity.py confirms the device build agrees."""
from __future__ import annotations

import ctypes
import json
import random
import struct
import subprocess
from pathlib import Path

import pytest

import corpus

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
LIB = ROOT / "tests" / "native" / "_build" / "libhostparse.so"


class HPRec(ctypes.Structure):
    _fields_ = [("epoch_sec", ctypes.c_int64), ("latitude", ctypes.c_double),
                ("longitude", ctypes.c_double), ("speed", ctypes.c_double),
                ("heading", ctypes.c_double), ("id_begin", ctypes.c_int32),
                ("id_len", ctypes.c_int32), ("postal_begin", ctypes.c_int32),
                ("postal_len", ctypes.c_int32)]


@pytest.fixture(scope="module")
def hp():
    srcs = [LIB.parents[1] / "hostparse.cpp"] + list((ROOT / "paper_2305_07454_b200" / "csrc").glob("*.cuh"))
    if not LIB.exists() or LIB.stat().st_mtime < max(s.stat().st_mtime for s in srcs):
        LIB.parent.mkdir(exist_ok=True)
        subprocess.run(["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-ffp-contract=off",
                        str(LIB.parents[1] / "hostparse.cpp"), "-o", str(LIB)], check=True)
    lib = ctypes.CDLL(str(LIB))
    lib.hp_parse_record.argtypes = [ctypes.c_char_p, ctypes.c_int32, ctypes.c_void_p,
                                    ctypes.POINTER(HPRec)]
    lib.hp_parse_header.argtypes = [ctypes.c_char_p, ctypes.c_int32, ctypes.c_void_p]
    lib.hp_parse_double.argtypes = [ctypes.c_char_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_double)]
    lib.hp_parse_timestamp.argtypes = [ctypes.c_char_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64)]
    lib.hp_cell_code.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_double,
                                 ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                 ctypes.c_double]
    lib.hp_cell_code.restype = ctypes.c_uint32
    lib.hp_extent_bins.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double]
    lib.hp_extent_bins.restype = ctypes.c_uint32
    return lib


def bits(x: float) -> str:
    return "%016x" % struct.unpack("<Q", struct.pack("<d", x))[0]


def from_bits(h: str) -> float:
    return struct.unpack("<d", struct.pack("<Q", int(h, 16)))[0]


CANON = (ctypes.c_int32 * 8)(0, 1, 2, 3, 4, 5, 6, 7)


def test_parse_kat(hp):
    bad = []
    for e in json.loads((GOLDEN / "parse_kat.json").read_text()):
        ln = e["line"].encode("latin-1")
        r = HPRec()
        why = hp.hp_parse_record(ln, len(ln), CANON, ctypes.byref(r))
        if why != e["reason"]:
            bad.append(("reason", e["line"], e["reason"], why))
            continue
        if why == -1:
            got = (r.epoch_sec, bits(r.latitude), bits(r.longitude), bits(r.speed), bits(r.heading),
                   ln[r.id_begin:r.id_begin + r.id_len].decode("latin-1").split("\0")[0],
                   ln[r.postal_begin:r.postal_begin + r.postal_len].decode("latin-1"))
            exp = (e["epoch"], e["lat"], e["lon"], e["speed"], e["heading"], e["id"], e["postal"])
            if got != exp:
                bad.append(("value", e["line"], exp, got))
    assert not bad, bad[:10]


def test_numeric_kat(hp):
    bad = []
    for e in json.loads((GOLDEN / "numeric_kat.json").read_text()):
        s = e["s"].encode("utf-8")
        out = ctypes.c_double()
        ok = hp.hp_parse_double(s, len(s), ctypes.byref(out))
        if e["bits"] is None:
            if ok:
                bad.append((e["s"], None, bits(out.value)))
        elif not ok:
            bad.append((e["s"], e["bits"], None))
        else:
            v = out.value
            if not (bits(v) == e["bits"] or (v != v and from_bits(e["bits"]) != from_bits(e["bits"]))):
                bad.append((e["s"], e["bits"], bits(v)))
    assert not bad, bad[:10]


def test_timestamp_kat(hp):
    for e in json.loads((GOLDEN / "timestamp_kat.json").read_text()):
        s = e["ts"].encode()
        out = ctypes.c_int64()
        ok = hp.hp_parse_timestamp(s, len(s), ctypes.byref(out))
        assert (out.value if ok else None) == e["epoch"], e


def test_header_kat(hp):
    for e in json.loads((GOLDEN / "header_kat.json").read_text()):
        h = e["header"].encode("latin-1")
        cols = (ctypes.c_int32 * 8)()
        ok = hp.hp_parse_header(h, len(h), cols)
        assert (list(cols) if ok else None) == e["cols"], e


def test_grid_kat(hp):
    """lat/lon/dxn/time bins through the fused cell_code against the reference bins."""
    for e in json.loads((GOLDEN / "grid_kat.json").read_text()):
        g = e["grid"]
        gd = (ctypes.c_double * 7)(g["lat_min"], g["lat_max"], g["lon_min"], g["lon_max"],
                                   g["lat_step"], g["lon_step"], g["dxn_offset"])
        gi = (ctypes.c_uint32 * 2)(g["min_step"], g["dxn_step"])
        R = hp.hp_extent_bins(g["lat_min"], g["lat_max"], g["lat_step"])
        C = hp.hp_extent_bins(g["lon_min"], g["lon_max"], g["lon_step"])
        assert (R, C) == (e["rows"], e["cols"])
        D = 360 // g["dxn_step"]
        mid_lat = g["lat_min"]
        mid_lon = g["lon_min"]
        for kind, val, rc, out in e["cases"]:
            if kind == "time":
                code = hp.hp_cell_code(gd, gi, 1, 250.0, val, mid_lat, mid_lon, 1.0, 0.0)
                assert rc == 0 and code // (D * R * C) == out, (g, val)
                continue
            x = from_bits(val)
            if kind == "lat":
                code = hp.hp_cell_code(gd, gi, 0, 250.0, 0, x, mid_lon, 1.0, 0.0)
                if rc:
                    assert code == 0x7FFFFFFC  # OutOfBounds when kept (require_in_grid=false)
                else:
                    assert (code // C) % R == out, (g, x)
            elif kind == "lon":
                code = hp.hp_cell_code(gd, gi, 0, 250.0, 0, mid_lat, x, 1.0, 0.0)
                if rc:
                    assert code == 0x7FFFFFFC
                else:
                    assert code % C == out, (g, x)
            elif kind == "dxn":
                code = hp.hp_cell_code(gd, gi, 1, 250.0, 0, mid_lat, mid_lon, 1.0, x)
                assert rc == 0 and (code // (R * C)) % D == out, (g, x)


def test_published_grid_kats(hp):
    # proj/tests/test_grid.cpp:63-117 and python/tests/test_smoke.py:21-30
    gd = (ctypes.c_double * 7)(36.0, 38.0, -93.0, -92.0, 0.01, 0.01, 0.0)
    gi = (ctypes.c_uint32 * 2)(5, 90)
    R, C = 200, 100
    code = hp.hp_cell_code(gd, gi, 1, 250.0, 18756 * 86400 + 3 * 3600 + 48 * 60 + 42, 37.664087,
                           -92.6546, 1.0, 33.0)
    t, rest = divmod(code, 4 * R * C)
    d, rest = divmod(rest, R * C)
    r, c = divmod(rest, C)
    assert (t, d, r, c) == (45, 0, 166, 34)


def test_filter_codes(hp):
    gd = (ctypes.c_double * 7)(36.0, 40.6, -95.8, -89.1, 0.1, 0.1, 0.0)
    gi = (ctypes.c_uint32 * 2)(5, 90)
    assert hp.hp_cell_code(gd, gi, 1, 250.0, 0, 35.0, -92.0, 10.0, 0.0) == 0x7FFFFFFF  # OutOfGrid
    assert hp.hp_cell_code(gd, gi, 1, 250.0, 0, 37.0, -92.0, 300.0, 0.0) == 0x7FFFFFFE  # Speed
    assert hp.hp_cell_code(gd, gi, 1, 250.0, 0, 37.0, -92.0, 250.0, 0.0) < 0x7FFFFFF0  # strict >


def test_differential_fuzz_vs_reference(hp, ref):
    """Fresh random corpus straight against the compiled reference (skipped without oracle/_ref)."""
    rng = random.Random(4242)
    cols = [0, 1, 2, 3, 4, 5, 6, 7]
    bad = 0
    for ln in corpus.line_corpus(rng, 4000):
        why, rec = ref.parse_record(ln, cols)
        r = HPRec()
        hw = hp.hp_parse_record(ln, len(ln), CANON, ctypes.byref(r))
        if why != hw:
            bad += 1
        elif why == -1 and (bits(rec.latitude), bits(rec.longitude), bits(rec.speed),
                            bits(rec.heading), rec.epoch_sec) != (
                bits(r.latitude), bits(r.longitude), bits(r.speed), bits(r.heading), r.epoch_sec):
            bad += 1
    for s in corpus.numeric_corpus(random.Random(99), 20000):
        b = s.encode("utf-8")
        v = ref.from_chars(b)
        out = ctypes.c_double()
        ok = hp.hp_parse_double(b, len(b), ctypes.byref(out))
        if (v is None) != (not ok) or (v is not None and v == v and bits(v) != bits(out.value)):
            bad += 1
    assert bad == 0
