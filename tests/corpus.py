"""Conformance corpus for record decode (SURVEY.md §7 hard part 1, §8(c)).

Lines / numeric fields / timestamps chosen to hit every branch of the reference's decode:
parse_record_impl (ingest.cpp:119-157), std::from_chars(double) via parse_double (:66-72),
Timestamp::parse (datetime.cpp:65-75), split_fields/trim (ingest.cpp:31-53).
"""
from __future__ import annotations

import random
import struct

NUMERIC_EDGE = [
    "37.664087", "-92.6546", "0", "-0", "0.0", "-0.0", "00037.5", "37.", ".5", "-.5", "1e1",
    "1E1", "1e+1", "1e-1", "3.7e1", "+1", "- 1", "0x1p3", "1_0", "1e", "1e+", "1e-", "e5", ".",
    "-", "-.", "inf", "-inf", "INF", "Infinity", "-infinity", "infinit", "nan", "NaN", "-nan",
    "nan()", "nan(abc_123)", "nan(", "nan(abc", "nan(a-b)", "+inf", "1e400", "1e-400", "1e-310",
    "4.9e-324", "2.4703282292062327e-324", "2.4703282292062328e-324", "5e-324", "3e-324",
    "1.7976931348623157e308", "1.7976931348623158e308", "1.7976931348623159e308", "1.8e308",
    "2.2250738585072011e-308", "2.2250738585072014e-308", "2.2250738585072012e-308",
    "37.66408700000000000000000000001", "359.999999999999999", "360", "360.0", "359.99",
    "-90", "90", "90.0000000000001", "-180", "180", "180.00001", "250", "250.0000001",
    "9007199254740993", "9007199254740992", "9007199254740991", "18446744073709551616",
    "123456789012345678901234567890", "0.1", "0.2", "0.3", "1e22", "1e23", "1e-22", "1e-23",
    "0.000000000000000000000000000001", "1" + "0" * 400, "0." + "0" * 400 + "1",
    "7.2057594037927933e16", "1.00000000000000011102230246251565404236316680908203125",
    "1.00000000000000011102230246251565404236316680908203124",
    "1.00000000000000011102230246251565404236316680908203126",
    "0e999999999999", "1e999999999999", "1e-999999999999", "123.456e-2", "12.34e5",
    " 1", "1 ", "1\t", "\t1", "1\r", "1..2", "1.2.3", "--1", "1-", "١",
    "100000000000000000000000", "8.98846567431158e307", "4.4501477170144023e-308",
]


def _rand_double_text(rng: random.Random) -> str:
    kind = rng.randrange(10)
    if kind == 0:
        return repr(rng.uniform(-200, 400))
    if kind == 1:
        return "%.17g" % rng.uniform(-200, 400)
    if kind == 2:
        x = struct.unpack("<d", struct.pack("<Q", rng.getrandbits(64)))[0]
        return "%.17g" % x
    if kind == 3:
        return "%.6f" % rng.uniform(-100, 100)
    if kind == 4:
        return "%.2f" % rng.uniform(0, 400)
    if kind == 5:
        return "%de%d" % (rng.randrange(1, 10 ** rng.randrange(1, 20)), rng.randrange(-340, 320))
    if kind == 6:  # near-halfway: 17-20 digits
        return "%d.%0*d" % (rng.randrange(0, 400), rng.randrange(15, 25),
                            rng.randrange(0, 10 ** 15))
    if kind == 7:
        return rng.choice(NUMERIC_EDGE)
    if kind == 8:
        return "%.3e" % rng.uniform(-1e10, 1e10)
    return "".join(rng.choice("0123456789.-+eE") for _ in range(rng.randrange(1, 8)))


TIMESTAMP_EDGE = [
    "2021-05-09 03:48:42", "2021-05-09T03:48:42", "2021-05-09 03:48", "2021-13-09 03:48:42",
    "2021-02-30 03:48:42", "2021-05-09 24:00:00", "2021-05-09 03:48:60", "", "2020-02-29 00:00:00",
    "2021-02-29 00:00:00", "2000-02-29 00:00:00", "1900-02-29 00:00:00", "0000-01-01 00:00:00",
    "1969-12-31 23:59:59", "1970-01-01 00:00:00", "9999-12-31 23:59:59", "2021-5-9 03:48:42",
    "2021-05-09  3:48:42", "2021-05-09 3:48:42", "2021-00-09 03:48:42", "2021-05-00 03:48:42",
    "2021-05-09 03:48:4a", "2021/05/09 00:00:00", " 2021-05-09 03:48:42", "2021-05-09 03:48:42 ",
    "2021-04-31 00:00:00", "2021-04-30 23:59:59", "1600-02-29 12:00:00", "2100-02-29 12:00:00",
]


def line_corpus(rng: random.Random, n_random: int = 2000) -> list[bytes]:
    """Whole data lines for the canonical 7-column header."""
    lines = [
        b"33456rd,2021-05-09 03:48:42,37.664087,-92.6546,65536,105.98,33",
        b"31224tf,2021-05-09 03:49:42,37.667707,-92.6490,65536,0,53",
        b"a,2021-05-09 00:00:00,37.0,-92.0,65536,10,360",
        b"a,2021-05-09 00:00:00,37.0,-92.0,65536,-5,33",
        b"a,2021-05-09 00:00:00,37.0,-92.0,65536,10,361",
        b"a,2021-05-09 00:00:00,95.0,-92.0,65536,10,33",
        b"a,2021-05-09 00:00:00,37.0,-192.0,65536,10,33",
        b"a,2021/05/09 00:00:00,37.0,-92.0,65536,10,33",
        b"a,2021-05-09 00:00:00,abc,-92.0,65536,10,33",
        b"a,2021-05-09 00:00:00,37.0,-92.0,65536,10",
        b",2021-05-09 00:00:00,37.0,-92.0,65536,10,33",
        b"bad line with,no real,fields,1,2,3,4",
        b"  j1 , 2021-05-09 00:00:00 ,\t37.5\t, -92.5 ,65101, 12.5 , 45 ",
        b"j1,2021-05-09 00:00:00,37.5,-92.5,,12.5,45",
        b"j1,2021-05-09 00:00:00,37.5,-92.5,65101,12.5,45,extra,cols",
        b"j1,2021-05-09 00:00:00,37.5,-92.5,65101,12.5,45,",
        b"   ",
        b"\r",
        b"j1,,37.5,-92.5,65101,12.5,45",
        b"j1,2021-05-09 00:00:00,inf,-92.5,65101,12.5,45",
        b"j1,2021-05-09 00:00:00,37.5,-92.5,65101,inf,45",
        b"j1,2021-05-09 00:00:00,37.5,-92.5,65101,nan,45",
        b"j1,2021-05-09 00:00:00,37.5,-92.5,65101,12.5,nan",
        b"j1,2021-05-09 00:00:00,37.5,-92.5,65101,12.5,-0",
        b"j1,2021-05-09 00:00:00,37.5,-92.5,65101,12.5,359.999999999999999",
        b"j1,2021-05-09 00:00:00,1e400,-92.5,65101,12.5,45",
        b"j1,2021-05-09 00:00:00,37.5,-92.5,65101,1e-400,45",
        b"j1,2021-05-09 00:00:00,37.5,-92.5,65101,-0.0,45",
        b"j1,2021-05-09 24:00:00,37.5,-92.5,65101,12.5,45",
        b"\xc3\xa9t\xc3\xa9,2021-05-09 00:00:00,37.5,-92.5,65101,12.5,45",
        b"j\x00x,2021-05-09 00:00:00,37.5,-92.5,65101,12.5,45",
    ]
    for s in NUMERIC_EDGE:
        lines.append(b"j9,2021-05-09 01:02:03,%s,-92.5,65101,12.5,45" % s.encode())
        lines.append(b"j9,2021-05-09 01:02:03,37.5,-92.5,65101,%s,45" % s.encode())
        lines.append(b"j9,2021-05-09 01:02:03,37.5,-92.5,65101,12.5,%s" % s.encode())
    for ts in TIMESTAMP_EDGE:
        lines.append(b"j8,%s,37.5,-92.5,65101,12.5,45" % ts.encode())
    for _ in range(n_random):
        f = [
            rng.choice(["j%06d" % rng.randrange(10 ** 6), "", " x ", "j" * rng.randrange(1, 40)]),
            rng.choice(TIMESTAMP_EDGE) if rng.random() < 0.2 else
            "2021-%02d-%02d %02d:%02d:%02d" % (rng.randrange(1, 13), rng.randrange(1, 29),
                                             rng.randrange(24), rng.randrange(60), rng.randrange(60)),
            _rand_double_text(rng), _rand_double_text(rng), rng.choice(["65101", "", " 7 "]),
            _rand_double_text(rng), _rand_double_text(rng),
        ]
        if rng.random() < 0.05:
            f = f[: rng.randrange(len(f))]
        if rng.random() < 0.05:
            f.append("extra")
        lines.append(",".join(f).encode())
    return lines


def numeric_corpus(rng: random.Random, n_random: int = 20000) -> list[str]:
    out = list(NUMERIC_EDGE)
    for _ in range(n_random):
        out.append(_rand_double_text(rng))
    return out


HEADER_CORPUS = [
    b"Journey Id,Timestamp,Latitude,Longitude,Postal Code,Speed,Heading",
    b"journey_id,timestamp,latitude,longitude,postal_code,speed,heading",
    b"JOURNEYID,TIMESTAMP,LATITUDE,LONGITUDE,POSTALCODE,SPEED,HEADING",
    b"Journey Id,Timestamp,Latitude,Longitude,Altitude,Postal Code,Speed,Heading",
    b"Journey Id,Timestamp,Latitude,Longitude,Postal Code,Speed",
    b"",
    b"heading,speed,zip code,longitude,latitude,timestamp,journey-id",
    b"Journey Id,Timestamp,Latitude,Longitude,Speed,Heading",
    b"Journey Id,Timestamp,Latitude,Longitude,Speed,Heading,Speed",
    b" Journey\tId ,Time_Stamp,LAT-itude,longitude,postalcode,speed\r,heading",
    b"nope,nope",
    b"Journey Id,Timestamp,Latitude,Longitude,Postal Code,Speed,Heading,Journey Id",
    b"journeyidx,timestamp,latitude,longitude,speed,heading",
]
