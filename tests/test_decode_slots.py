"""Per-line device decode parity (SURVEY section 8(c) parity plan (i)): for every data line the
GPU decode (K1, read back through cvlg_debug_slots) agrees with the UNMODIFIED reference
parse_record_impl (ingest.cpp:119-157, via oracle/_ref) — accepted vs rejected, epoch seconds,
the f64 speed bit pattern — and its cell code equals the reference's bins
(lat_bin/lon_bin/time_bin/dxn_bin/global_index, grid.cpp:10-90) and filter verdict
(filter_reason, aggregate.cpp:48-56). Lines: the golden parse KATs (tests/golden/parse_kat.json,
generated from the reference), the malformed-line corpus and synthetic rows; both canonical
order paths (run-merge fast path and the full-sort path)."""
from __future__ import annotations

import ctypes
import json
import random
import struct
from pathlib import Path

import numpy as np
import pytest

from helpers import HEADER, write_shards

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
K_REJECTED, K_OOG, K_SPEED, K_UNBINNABLE = 0x7FFFFFFB, 0x7FFFFFFF, 0x7FFFFFFE, 0x7FFFFFFC


def slots(ctx):
    import paper_2305_07454_b200 as cvlg
    lib = cvlg.cvlg.lib()
    lib.cvlg_debug_slots.argtypes = [ctypes.c_void_p] * 5 + [ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64)]
    n = ctypes.c_uint64()
    cvlg.cvlg._check(lib.cvlg_debug_slots(ctx.handle, None, None, None, None, 0, ctypes.byref(n)))
    N = n.value
    ts = np.zeros(N, np.int64)
    sp = np.zeros(N, np.float64)
    code = np.zeros(N, np.uint32)
    loff = np.zeros(N, np.uint64)
    cvlg.cvlg._check(lib.cvlg_debug_slots(ctx.handle, ts.ctypes.data_as(ctypes.c_void_p),
                                          sp.ctypes.data_as(ctypes.c_void_p),
                                          code.ctypes.data_as(ctypes.c_void_p),
                                          loff.ctypes.data_as(ctypes.c_void_p), N, ctypes.byref(n)))
    return ts, sp, code, loff


def expected_code(ref, spec, rec):
    inside = spec.lat_min <= rec.latitude <= spec.lat_max and spec.lon_min <= rec.longitude <= spec.lon_max
    if not inside:
        return K_OOG
    if rec.speed > 250.0:
        return K_SPEED
    T, D, R, C = spec.dims()
    r = ref.bin(spec, 0, rec.latitude)[1]
    c = ref.bin(spec, 1, rec.longitude)[1]
    t = ref.bin(spec, 2, 0.0, rec.epoch_sec)[1]
    d = ref.bin(spec, 3, rec.heading)[1]
    return ((t * D + d) * R + r) * C + c


def check(ref, paths, spec):
    import paper_2305_07454_b200 as cvlg
    ctx = cvlg.Context()
    cvlg.run_pipeline(paths, spec, ctx=ctx)
    ts, sp, code, loff = slots(ctx)
    blob = b"".join(Path(p).read_bytes() for p in sorted(paths))
    cols = ref.parse_header(HEADER)
    n_lines = 0
    for i in range(len(ts)):
        a = int(loff[i])
        e = blob.find(b"\n", a)
        line = blob[a: e if e >= 0 else len(blob)]
        if line.endswith(b"\r"):
            line = line[:-1]
        if not line:
            continue  # "\r\n": an inert slot, not a row (ingest.cpp:227)
        n_lines += 1
        why, rec = ref.parse_record(line, cols)
        got = int(code[i]) & 0x7FFFFFFF
        if why != -1:
            assert got == K_REJECTED, (line, why, hex(got))
            continue
        assert got != K_REJECTED, (line, hex(got))
        assert int(ts[i]) == rec.epoch_sec, (line, int(ts[i]), rec.epoch_sec)
        assert struct.pack("<d", float(sp[i])) == struct.pack("<d", rec.speed), (line, sp[i], rec.speed)
        assert got == expected_code(ref, spec, rec), (line, hex(got), hex(expected_code(ref, spec, rec)))
    rows = sum(1 for p in paths for l in Path(p).read_bytes().split(b"\n")[1:]
               if (l[:-1] if l.endswith(b"\r") else l))  # one '\r' stripped (ingest.cpp:208)
    assert n_lines == rows
    ctx.close()
    return n_lines


def kat_lines():
    kat = json.loads((ROOT / "tests" / "golden" / "parse_kat.json").read_text())
    return [k["line"].encode("latin-1") for k in kat]


def test_decode_slots_golden_kat_and_corpus(ref, tmp_path):
    import corpus
    import paper_2305_07454_b200 as cvlg
    lines = kat_lines() + corpus.line_corpus(random.Random(21), 3000)
    lines = [l for l in lines if b"\n" not in l]
    # every line its own journey-ish mix -> many run heads -> the full-sort path
    contents = [HEADER + b"\n" + b"\n".join(lines[0::2]) + b"\n",
                HEADER + b"\r\n" + b"\r\n".join(lines[1::2])]
    paths = write_shards(tmp_path, contents)
    for spec in (cvlg.GridSpec(), cvlg.GridSpec(lat_step=0.013, lon_step=0.007, min_step=1, dxn_step=120, dxn_offset=45.0)):
        assert check(ref, paths, spec) > 4000


def test_decode_slots_synthetic_run_merge_path(ref, day_cache, tmp_path):
    import paper_2305_07454_b200 as cvlg
    paths, rows = day_cache(seed=61, journeys=60, shards=4)
    # plus a sprinkle of malformed lines inside the runs
    extra = tmp_path / "x"
    contents = []
    rng = random.Random(3)
    for p in paths:
        ls = Path(p).read_bytes().split(b"\n")
        body = [l for l in ls[1:] if l]
        for _ in range(20):
            k = rng.randrange(len(body))
            body.insert(k, rng.choice([b"j000001,2021-05-09 25:00:00,37.5,-92.5,65101,12.5,45",
                                       b"j000002,2021-05-09 01:00:00,abc,-92.5,65101,12.5,45",
                                       b"j000003,2021-05-09 01:00:00,37.5,-92.5,65101,999,45",
                                       b"j000004,2021-05-09 01:00:00,95.5,-92.5,65101,12.5,45"]))
        contents.append(ls[0] + b"\n" + b"\n".join(body) + b"\n")
    paths2 = write_shards(extra, contents)
    assert check(ref, paths2, cvlg.GridSpec()) > rows
