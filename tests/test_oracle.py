"""CPU tests (no GPU): pin the plain-C restatement oracle (oracle/cvl_oracle.c) against the golden
vectors generated from the compiled reference (tests/golden/make_golden.py) and the reference's
own published KATs (proj/tests/*.cpp), and — when oracle/_ref is built — against the reference
itself on synthetic days."""
from __future__ import annotations

import hashlib
import json
import struct
import tempfile
from pathlib import Path

import numpy as np
import pytest

from helpers import shuffle_rows

GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def ora():
    from oracle.oracle import Restated
    if not Restated.available():
        pytest.skip("oracle/_build not built")
    return Restated()


def bits(x: float) -> str:
    return "%016x" % struct.unpack("<Q", struct.pack("<d", x))[0]


class G:  # GridSpec stand-in for the oracle helpers
    def __init__(self, d):
        self.__dict__.update(d)


def test_numeric_kat(ora):
    bad = []
    for e in json.loads((GOLDEN / "numeric_kat.json").read_text()):
        v = ora.parse_double(e["s"].encode("utf-8"))
        got = None if v is None else bits(v)
        if e["bits"] is None:
            ok = got is None
        else:
            # NaN payloads are irrelevant downstream (always RangeViolation)
            ok = got is not None and (got == e["bits"] or (v != v and e["bits"][1:4] in ("ff8", "ff0")))
        if not ok:
            bad.append((e["s"], e["bits"], got))
    assert not bad, bad[:10]


def test_timestamp_kat(ora):
    for e in json.loads((GOLDEN / "timestamp_kat.json").read_text()):
        assert ora.parse_timestamp(e["ts"].encode()) == e["epoch"], e


def test_datetime_published_kats(ora):
    # proj/tests/test_datetime.cpp:7-50
    assert ora.parse_timestamp(b"2021-05-09 03:48:42") == 18756 * 86400 + 3 * 3600 + 48 * 60 + 42
    assert ora.parse_timestamp(b"2020-02-29 00:00:00") is not None
    assert ora.parse_timestamp(b"2021-02-29 00:00:00") is None
    assert ora.parse_timestamp(b"1900-02-29 00:00:00") is None
    assert ora.parse_timestamp(b"2000-02-29 00:00:00") is not None
    assert ora.parse_timestamp(b"1969-12-31 23:59:59") == -1


def test_header_kat(ora):
    for e in json.loads((GOLDEN / "header_kat.json").read_text()):
        assert ora.parse_header(e["header"].encode("latin-1")) == e["cols"], e


def test_journey_hash(ora):
    # FNV-1a 64 (ingest.cpp:287-291) offset basis / prime
    assert ora.journey_hash(b"") == 1469598103934665603
    for s in [b"a", b"j000001", b"33456rd", b"vehicle-000000000001"]:
        h = 1469598103934665603
        for c in s:
            h = ((h ^ c) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
        assert ora.journey_hash(s) == h


@pytest.mark.parametrize("case", ["synth_small", "dups_shuffled", "malformed", "table1"])
def test_golden_days(ora, case):
    d = GOLDEN / "days" / case
    meta = json.loads((d / "expected.json").read_text())
    exp = np.load(d / "expected.npz")
    paths = [str(d / s) for s in meta["shards"]]
    planes, raw, st = ora.run_pipeline(paths, G(meta["grid"]))
    assert np.array_equal(planes, exp["planes"])
    assert np.array_equal(raw, exp["raw"])
    assert st == meta["stats"]
    with tempfile.TemporaryDirectory() as t:
        p = Path(t) / "x.cvl1"
        import ctypes
        from oracle.oracle import grid_struct
        n = ctypes.c_uint64()
        rc = ora.lib.ora_write_container(planes.ctypes.data_as(ctypes.c_void_p),
                                         ctypes.byref(grid_struct(G(meta["grid"]))), 18756,
                                         str(p).encode(), ctypes.byref(n))
        assert rc == 0
        assert hashlib.sha256(p.read_bytes()).hexdigest() == meta["container_sha256_day18756"]


def test_table1_published_values(ora):
    # acceptance.cpp:247-293: dedup 4->3, volume 3, mean 51.45333 (+-1e-5), t=45, d=0
    d = GOLDEN / "days" / "table1"
    meta = json.loads((d / "expected.json").read_text())
    planes, raw, st = ora.run_pipeline([str(d / "shard_0000.csv")], G(meta["grid"]))
    assert st["duplicates_dropped"] == 1 and st["accepted"] == 3
    assert planes[45, 4, 0, 0] == 3
    assert abs(float(planes[45, 0, 0, 0:1].view(np.float32)[0]) - 51.45333) < 1e-5
    assert raw[45, 0, 0, 0] == 3


def test_container_size_law(ora, tmp_path):
    # acceptance.cpp:200-244: 10 x 20 grid -> 58 + 288 * (4 + 8 * 200 * 4) = 1,844,410 bytes
    import ctypes
    from oracle.oracle import grid_struct
    g = G(dict(lat_min=36.0, lat_max=36.1, lon_min=-93.0, lon_max=-92.8, lat_step=0.01,
               lon_step=0.01, min_step=5, dxn_step=90, dxn_offset=0.0))
    assert ora.dims(g) == (288, 4, 10, 20)
    planes = np.zeros((288, 8, 10, 20), dtype=np.uint32)
    n = ctypes.c_uint64()
    assert ora.lib.ora_write_container(planes.ctypes.data_as(ctypes.c_void_p),
                                       ctypes.byref(grid_struct(g)), 18756,
                                       str(tmp_path / "c.cvl1").encode(), ctypes.byref(n)) == 0
    assert n.value == 1844410 == (tmp_path / "c.cvl1").stat().st_size


def test_restatement_matches_reference_on_synth_days(ora, ref, day_cache, tmp_path):
    """Differential pin against the compiled reference (skipped when oracle/_ref is absent)."""
    from oracle.oracle import CGrid  # noqa: F401
    specs = [G(dict(lat_min=36.0, lat_max=40.6, lon_min=-95.8, lon_max=-89.1, lat_step=s,
                    lon_step=s, min_step=m, dxn_step=90, dxn_offset=o))
             for s, m, o in [(0.1, 5, 0.0), (0.25, 60, 45.0), (10.0, 5, 0.0)]]
    for kw in [dict(seed=2, journeys=40), dict(seed=4, journeys=30, sample_period=0.5)]:
        paths, _ = day_cache(**kw)
        variants = [paths, shuffle_rows(paths, tmp_path / f"s{kw['seed']}", 4, seed=1)]
        for ps in variants:
            for spec in specs:
                a = ref.run_pipeline(ps, spec)
                b = ora.run_pipeline(ps, spec)
                assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
                assert a[2] == b[2]
