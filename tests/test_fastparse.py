"""CPU tests (no GPU) of K1's SWAR fast path (csrc/fastparse.cuh) compiled for the host: every
decision it takes must equal the general restatement of parse_record_impl (parse.cuh), which is
itself pinned to the reference (test_hostparse.py). The same header is compiled for sm_100a."""
from __future__ import annotations

import ctypes
import json
import random
from pathlib import Path

import numpy as np
import pytest

from test_hostparse import GOLDEN, hp  # noqa: F401  (fixture)


def _setup(lib):
    u64p = ctypes.POINTER(ctypes.c_uint64)
    lib.hp_fuzz_fast_number.restype = ctypes.c_uint64
    lib.hp_fuzz_fast_number.argtypes = [ctypes.c_uint64, ctypes.c_uint64, u64p, ctypes.c_char_p]
    lib.hp_fuzz_fast_number_hit.restype = ctypes.c_uint64
    lib.hp_fuzz_fast_number_hit.argtypes = [ctypes.c_uint64, ctypes.c_uint64, u64p, ctypes.c_char_p]
    lib.hp_fuzz_fast_timestamp.restype = ctypes.c_uint64
    lib.hp_fuzz_fast_timestamp.argtypes = lib.hp_fuzz_fast_number.argtypes
    lib.hp_fast_number.argtypes = [ctypes.c_char_p, ctypes.c_int32, ctypes.c_int, ctypes.c_int,
                                   ctypes.POINTER(ctypes.c_double)]
    lib.hp_fast_timestamp.argtypes = [ctypes.c_char_p, ctypes.c_int32, ctypes.c_int,
                                      ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_uint32)]
    lib.hp_time_bin_mod.restype = ctypes.c_uint32
    lib.hp_time_bin_mod.argtypes = [ctypes.c_uint32, ctypes.c_uint32]
    lib.hp_time_bin.restype = ctypes.c_uint32
    lib.hp_time_bin.argtypes = [ctypes.c_int64, ctypes.c_uint32]
    lib.hp_div_pow10.restype = ctypes.c_double
    lib.hp_div_pow10.argtypes = [ctypes.c_double, ctypes.c_int]
    return lib


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_fast_number_fuzz(hp, seed):
    lib = _setup(hp)
    d = ctypes.c_uint64()
    b = ctypes.create_string_buffer(64)
    bad = lib.hp_fuzz_fast_number(seed, 2_000_000, ctypes.byref(d), b)
    assert bad == 0, b.value
    assert d.value > 500_000  # the fast path decides most well-formed numbers


def test_fast_number_golden_fields(hp):
    """Every numeric KAT field of the reference (tests/golden/numeric_kat.json): when the fast
    path decides, it agrees with std::from_chars bit for bit; it must decide the synth shapes."""
    lib = _setup(hp)
    cases = json.loads((GOLDEN / "numeric_kat.json").read_text())
    v = ctypes.c_double()
    decided = 0
    for c in cases:
        s = c["s"].encode("utf-8", "surrogateescape")
        for shift in range(4):
            if lib.hp_fast_number(s, len(s), shift, -1, ctypes.byref(v)):
                decided += 1
                assert c.get("bits") is not None, s  # the reference accepts it
                got = "%016x" % np.float64(v.value).view(np.uint64)
                assert got == c["bits"], (s, got, c["bits"])
    assert decided > 0
    for s in [b"37.664087", b"-92.654600", b"78.36", b"359.99", b"0.00", b"7.5"]:
        assert lib.hp_fast_number(s, len(s), 0, -1, ctypes.byref(v)) == 1, s


def test_fast_timestamp_fuzz(hp):
    lib = _setup(hp)
    d = ctypes.c_uint64()
    b = ctypes.create_string_buffer(64)
    bad = lib.hp_fuzz_fast_timestamp(5, 2_000_000, ctypes.byref(d), b)
    assert bad == 0, b.value
    assert d.value > 200_000


def test_time_bin_from_minute(hp):
    """time_bin via the parsed minute and a multiply-high equals grid.cpp:69-71 for every minute
    and every legal min_step (divisors of 1440)."""
    lib = _setup(hp)
    steps = [s for s in range(1, 1441) if 1440 % s == 0]
    for st in steps:
        for minute in range(1440):
            assert lib.hp_time_bin_mod(minute, st) == lib.hp_time_bin(minute * 60 + 17, st)


def test_markstein_division(hp):
    """x / 10^k through RN(10^-k) + one FMA correction equals IEEE division (the exhaustive
    4.8e9-case sweep is tools/check_div.c; this samples it)."""
    lib = _setup(hp)
    rng = random.Random(11)
    xs = list(range(0, 20000)) + [rng.randrange(0, 10**12) for _ in range(60000)]
    for k in range(1, 9):
        p = 10.0 ** k
        for x in xs:
            assert lib.hp_div_pow10(float(x), k) == float(x) / p, (x, k)


def test_class_masks(hp):
    """K1's '\\n' / ',' bitmaps (multiply-gather compression) equal a byte loop."""
    hp.hp_check_class_masks.restype = ctypes.c_uint64
    hp.hp_check_class_masks.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
    assert hp.hp_check_class_masks(1, 3_000_000) == 0


def test_binning_fast_path(hp):
    """floor(snap(d / step)) via RN(d * RN(1/step)) with the 4e-9 edge guard equals the exact
    division + snap of grid.cpp:10-36, on quotients concentrated at and around bin edges."""
    hp.hp_fuzz_snapped_floor.restype = ctypes.c_uint64
    hp.hp_fuzz_snapped_floor.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int]
    steps = [0.1, 0.01, 0.013, 0.007, 0.25, 10.0, 90.0, 120.0, 45.0, 0.02, 1.0 / 3.0, 0.3]
    arr = (ctypes.c_double * len(steps))(*steps)
    assert hp.hp_fuzz_snapped_floor(1, 3_000_000, arr, len(steps)) == 0


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_fast_number_hit_fuzz(hp, seed):
    """K1's cached-shape number path (fast_number_hit) never disagrees with from_chars, and it
    decides a large share of the canonical shapes."""
    lib = _setup(hp)
    d = ctypes.c_uint64()
    b = ctypes.create_string_buffer(64)
    bad = lib.hp_fuzz_fast_number_hit(seed, 400_000, ctypes.byref(d), b)
    assert bad == 0, b.value
    assert d.value > 50_000
