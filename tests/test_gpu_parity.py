"""GPU parity: the sm_100a pipeline (through the C ABI) against the UNMODIFIED reference
cvl::run_pipeline (oracle/_ref) on the same shard files. Bar: bit-identical speed bits, volumes,
raw counts and identical PipelineStats (SURVEY §8c parity plan iii/iv)."""
from __future__ import annotations

import random
from pathlib import Path

import numpy as np
import pytest

from helpers import HEADER, commuter_days, diff_lattice, shuffle_rows, stats_dict, write_shards

pytestmark = pytest.mark.gpu


def run_both(ref, paths, spec, rules=None, partitions=3):
    import paper_2305_07454_b200 as cvlg
    ep, er, est, _ = ref.run_pipeline(paths, spec, rules, n_partitions=partitions, n_threads=1)
    st = cvlg.PipelineStats()
    lat = cvlg.run_pipeline(paths, spec, rules or cvlg.FilterRules(), n_partitions=partitions,
                            stats=st)
    return (ep, er, est), (lat.planes, lat.raw, stats_dict(st))


def assert_parity(ref, paths, spec, rules=None):
    (ep, er, est), (gp, gr, gst) = run_both(ref, paths, spec, rules)
    d = diff_lattice(ep, er, gp, gr)
    assert d == "", d
    assert gst == est
    return est


def spec_default():
    import paper_2305_07454_b200 as cvlg
    return cvlg.GridSpec()


def spec_coarse():
    import paper_2305_07454_b200 as cvlg
    return cvlg.GridSpec(lat_step=0.25, lon_step=0.25)


def spec_degenerate():
    import paper_2305_07454_b200 as cvlg
    return cvlg.GridSpec(lat_step=10.0, lon_step=10.0)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_synth_day_default_grid(ref, day_cache, seed):
    paths, rows = day_cache(seed=seed, journeys=120, mean_duration=300.0)
    est = assert_parity(ref, paths, spec_default())
    assert est["rows_read"] == rows and est["accepted"] == rows


@pytest.mark.parametrize("grid", ["coarse", "degenerate"])
def test_acceptance_grids(ref, day_cache, grid):
    # acceptance.cpp:130-159 grids
    paths, _ = day_cache(seed=7, journeys=150, mean_duration=240.0)
    assert_parity(ref, paths, spec_coarse() if grid == "coarse" else spec_degenerate())


def test_grid_variants(ref, day_cache):
    import paper_2305_07454_b200 as cvlg
    paths, _ = day_cache(seed=11, journeys=80)
    for spec in [cvlg.GridSpec(min_step=60), cvlg.GridSpec(dxn_offset=45.0),
                 cvlg.GridSpec(dxn_step=180, min_step=1440), cvlg.GridSpec(dxn_step=360),
                 cvlg.GridSpec(lat_step=0.013, lon_step=0.007, min_step=1),
                 cvlg.GridSpec(lat_min=37.0, lat_max=38.0, lon_min=-93.0, lon_max=-92.0,
                               lat_step=0.01, lon_step=0.01),
                 cvlg.GridSpec(dxn_step=120, dxn_offset=-30.0)]:
        assert_parity(ref, paths, spec)


def test_duplicates_slow_path(ref, day_cache):
    # sample_period 0.5 renders duplicate (journey, second) keys (test_synth.cpp:104-140)
    paths, _ = day_cache(seed=5, journeys=60, sample_period=0.5)
    est = assert_parity(ref, paths, spec_default())
    assert est["duplicates_dropped"] > 0


def test_shuffled_rows(ref, day_cache, tmp_path):
    paths, _ = day_cache(seed=9, journeys=100)
    sh = shuffle_rows(paths, tmp_path / "sh", 7, seed=3)
    assert_parity(ref, sh, spec_default())
    assert_parity(ref, sh, spec_degenerate())


def test_shuffled_with_dups(ref, day_cache, tmp_path):
    paths, _ = day_cache(seed=5, journeys=60, sample_period=0.5)
    sh = shuffle_rows(paths, tmp_path / "sh", 5, seed=4)
    est = assert_parity(ref, sh, spec_default())
    assert est["duplicates_dropped"] > 0


def test_manifest_order_and_partitions(ref, day_cache):
    import paper_2305_07454_b200 as cvlg
    paths, _ = day_cache(seed=2, journeys=90)
    base = cvlg.run_pipeline(paths, spec_coarse(), n_partitions=1)
    shuffled = list(paths)
    random.Random(13).shuffle(shuffled)
    for parts in (2, 4, 16):
        other = cvlg.run_pipeline(shuffled, spec_coarse(), n_partitions=parts)
        assert np.array_equal(base.planes, other.planes)
    ep, _, _, _ = ref.run_pipeline(shuffled, spec_coarse(), n_partitions=4)
    assert np.array_equal(ep, base.planes)


def test_table1_rows(ref, tmp_path):
    # acceptance.cpp:247-293 golden rows (dedup 4->3, volume 3, mean 51.45333)
    rows = [
        b"33456rd,2021-05-09 03:48:42,37.664087,-92.6546,65536,105.98,33",
        b"31224tf,2021-05-09 03:49:42,37.667707,-92.6490,65536,0,53",
        b"22124fs,2021-05-09 03:49:49,37.690978,-92.6490,65536,48.38,33",
        b"33456rd,2021-05-09 03:48:42,37.664087,-92.6546,65536,105.98,33",
    ]
    paths = write_shards(tmp_path, [HEADER + b"\n" + b"\n".join(rows) + b"\n"])
    est = assert_parity(ref, paths, spec_degenerate())
    assert est["duplicates_dropped"] == 1 and est["accepted"] == 3
    import paper_2305_07454_b200 as cvlg
    lat = cvlg.run_pipeline(paths, spec_degenerate())
    assert lat.volume[45, 0, 0, 0] == 3
    assert abs(float(lat.speed[45, 0, 0, 0]) - 51.45333) < 1e-5


def test_malformed_and_edge_inputs(ref, tmp_path):
    from helpers import malformed_contents
    paths = write_shards(tmp_path, malformed_contents(5))
    for spec in (spec_default(), spec_degenerate()):
        est = assert_parity(ref, paths, spec)
    assert est["rejected"].get("BadHeader") == 1
    assert sum(est["rejected"].values()) > 100


def test_long_and_unusual_ids(ref, tmp_path):
    rng = random.Random(8)
    ids = (["vehicle-%012d" % i for i in range(40)] + ["j%07d" % i for i in range(999990, 1000010)]
           + ["x" * n for n in range(1, 20)] + ["é%d" % i for i in range(5)]
           + ["a\tb", "ab", "ab\x00", "ab\x00\x00", "\xff\xfe", "\x7f" * 16, "q" * 300])
    lines = []
    for k in range(6000):
        jid = rng.choice(ids).encode("latin-1")
        lines.append(b"%s,2021-05-09 %02d:%02d:%02d,%.6f,%.6f,65101,%.2f,%.2f" % (
            jid, rng.randrange(24), rng.randrange(60), rng.randrange(60),
            rng.uniform(36.0, 40.6), rng.uniform(-95.8, -89.1), rng.uniform(0, 140),
            rng.uniform(0, 360)))
    paths = write_shards(tmp_path, [HEADER + b"\n" + b"\n".join(lines[i::3]) + b"\n"
                                    for i in range(3)])
    for spec in (spec_default(), spec_degenerate()):
        assert_parity(ref, paths, spec)


def test_filters(ref, day_cache, tmp_path):
    import paper_2305_07454_b200 as cvlg
    paths, _ = day_cache(seed=4, journeys=80)
    narrow = cvlg.GridSpec(lat_min=37.0, lat_max=39.0, lon_min=-94.0, lon_max=-91.0)
    est = assert_parity(ref, paths, narrow)
    assert est["filtered"]["OutOfGrid"] > 0
    est = assert_parity(ref, paths, spec_default(), cvlg.FilterRules(speed_ceiling=80.0))
    assert est["filtered"]["SpeedCeiling"] > 0


def test_out_of_bounds_error(day_cache):
    import paper_2305_07454_b200 as cvlg
    paths, _ = day_cache(seed=4, journeys=40)
    narrow = cvlg.GridSpec(lat_min=37.0, lat_max=39.0, lon_min=-94.0, lon_max=-91.0)
    with pytest.raises(cvlg.CvlError) as e:
        cvlg.run_pipeline(paths, narrow, cvlg.FilterRules(require_in_grid=False))
    assert e.value.code == "OutOfBounds"


def test_multi_day_fold(ref, day_cache):
    # time_bin ignores the date (grid.cpp:69-71): two days fold onto one lattice
    a, _ = day_cache(seed=21, journeys=60, day="2021-05-09")
    b, _ = day_cache(seed=21, journeys=60, day="2021-05-10")
    c, _ = day_cache(seed=22, journeys=60, day="2021-05-11")
    assert_parity(ref, a + b + c, spec_default())


def test_container_bytes(ref, day_cache, tmp_path):
    import paper_2305_07454_b200 as cvlg
    paths, _ = day_cache(seed=3, journeys=50)
    spec = spec_coarse()
    lat = cvlg.run_pipeline(paths, spec)
    ours = tmp_path / "ours.cvl1"
    theirs = tmp_path / "ref.cvl1"
    n = cvlg.write_container(lat, spec, 18756, ours)
    ep, _, _, _ = ref.run_pipeline(paths, spec)
    m = ref.write_container(ep, spec, 18756, theirs)
    assert n == m and ours.read_bytes() == theirs.read_bytes()


def test_host_and_device_entry_points(ref, day_cache):
    import torch
    import paper_2305_07454_b200 as cvlg
    paths, _ = day_cache(seed=6, journeys=70)
    spec = spec_default()
    ep, er, est, _ = ref.run_pipeline(sorted(paths), spec)
    bufs = [Path(p).read_bytes() for p in sorted(paths)]
    st = cvlg.PipelineStats()
    lat = cvlg.run_pipeline_host(bufs, spec, stats=st)
    assert diff_lattice(ep, er, lat.planes, lat.raw) == ""
    assert stats_dict(st) == est
    blob = b"".join(bufs)
    offs = [0]
    for b in bufs:
        offs.append(offs[-1] + len(b))
    d_csv = torch.frombuffer(bytearray(blob), dtype=torch.uint8).cuda()
    t, _, r, c = spec.dims()
    d_planes = torch.empty((t, 8, r, c), dtype=torch.int32, device="cuda")
    d_raw = torch.empty((t, 4, r, c), dtype=torch.int32, device="cuda")
    st2 = cvlg.PipelineStats()
    cvlg.run_pipeline_device(d_csv.data_ptr(), offs, d_planes.data_ptr(), d_raw.data_ptr(), spec,
                             stats=st2)
    torch.cuda.synchronize()
    gp = d_planes.cpu().numpy().view(np.uint32)
    gr = d_raw.cpu().numpy().view(np.uint32)
    assert diff_lattice(ep, er, gp, gr) == ""
    assert stats_dict(st2) == est


def test_cpp_dropin_with_reference_types(day_cache):
    """include/cvlg.hpp: cvl::gpu::run_pipeline over the reference's own C++ types, compared
    in C++ with cvl::run_pipeline (BatchFrame::bitwise_equal, raw counts, stats, container
    bytes) — tests/native/dropin_main.cpp."""
    import subprocess
    exe = Path(__file__).resolve().parent / "native" / "_build" / "dropin"
    if not exe.exists():
        pytest.skip("drop-in demo not built (needs the reference headers at build time)")
    paths, _ = day_cache(seed=12, journeys=50)
    for step in ("0.1", "0.25", "10"):
        r = subprocess.run([str(exe), step, *paths], capture_output=True, text=True)
        assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    golden = Path(__file__).resolve().parent / "golden" / "days" / "malformed"
    r = subprocess.run([str(exe), "0.5", *sorted(str(p) for p in golden.glob("*.csv"))],
                       capture_output=True, text=True)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)


def test_golden_days_gpu():
    """Committed reference fixtures (no reference needed at run time)."""
    import json
    import paper_2305_07454_b200 as cvlg
    root = Path(__file__).resolve().parent / "golden" / "days"
    for case in ("synth_small", "dups_shuffled", "malformed", "table1"):
        meta = json.loads((root / case / "expected.json").read_text())
        exp = np.load(root / case / "expected.npz")
        st = cvlg.PipelineStats()
        lat = cvlg.run_pipeline([str(root / case / s) for s in meta["shards"]],
                                cvlg.GridSpec(**meta["grid"]), stats=st)
        assert diff_lattice(exp["planes"], exp["raw"], lat.planes, lat.raw) == "", case
        assert stats_dict(st) == meta["stats"], case


def test_empty_manifest(ref):
    import paper_2305_07454_b200 as cvlg
    st = cvlg.PipelineStats()
    lat = cvlg.run_pipeline([], spec_default(), stats=st)
    ep, er, est, _ = ref.run_pipeline([], spec_default())
    assert diff_lattice(ep, er, lat.planes, lat.raw) == ""
    assert stats_dict(st) == est


def test_zero_partitions(day_cache):
    import paper_2305_07454_b200 as cvlg
    paths, _ = day_cache(seed=1, journeys=10)
    with pytest.raises(cvlg.CvlError) as e:
        cvlg.run_pipeline(paths, spec_default(), n_partitions=0)
    assert e.value.code == "ZeroPartitions"


def test_dense_short_lines_overflow_tiles(ref, tmp_path):
    """Tiles holding more than 384 data lines (lines averaging < 43 bytes) take K1's overflow
    slot region; mixed with long lines that cross the 16 KB tile boundary beyond the staged halo
    (general path over global memory) and blank / CRLF lines."""
    rng = random.Random(17)
    short = []
    for i in range(30000):  # "a,2021-05-09 HH:MM:SS,37,-92,1,5,9" ~ 34 bytes
        j = rng.randrange(40)
        short.append(b"%c%d,2021-05-09 %02d:%02d:%02d,%d.%d,-%d.%d,1,%d,%d" % (
            97 + j % 26, j, (i // 3600) % 24, (i // 60) % 60, i % 60, 36 + rng.randrange(4),
            rng.randrange(10), 90 + rng.randrange(5), rng.randrange(10), rng.randrange(130),
            rng.randrange(360)))
    longl = [b"L%03d,2021-05-09 10:%02d:%02d,37.123456789012345678901234567890123,-92.5%s,65101,12.5,45" % (
        k, k // 60, k % 60, b"0" * rng.randrange(60, 700)) for k in range(200)]
    lines = short + longl
    rng.shuffle(lines)
    blob_a = HEADER + b"\n" + b"\n".join(lines[:16000]) + b"\n"
    blob_b = HEADER + b"\r\n" + b"\r\n\r\n".join(lines[16000:]) + b"\r\n"
    paths = write_shards(tmp_path, [blob_a, blob_b])
    est = assert_parity(ref, paths, spec_default())
    assert est["rows_read"] == len(lines)
    assert_parity(ref, paths, spec_coarse())


def test_benchmark_workload_c2_bitexact(ref, tmp_path):
    """The bench workload itself (configs[1], c2: 100k journeys, seed 1, mean duration 500 s,
    16 shards, 49,977,768 rows, default grid): lattice bits, raw counts and statistics identical
    to cvl::run_pipeline (16 threads, 32 partitions) on the same shard files."""
    import os
    import paper_2305_07454_b200 as cvlg
    blob, offs, rows = cvlg.synth_day(seed=1, journeys=100_000, shards=16, mean_duration=500.0)
    assert rows == 49_977_768
    paths = write_shards(tmp_path, [blob[offs[i]:offs[i + 1]].tobytes() for i in range(16)])
    threads = max(1, min(16, os.cpu_count() or 1))
    ep, er, est, _ = ref.run_pipeline(paths, spec_default(), None, n_partitions=2 * threads,
                                      n_threads=threads)
    st = cvlg.PipelineStats()
    lat = cvlg.run_pipeline(paths, spec_default(), stats=st)
    d = diff_lattice(ep, er, lat.planes, lat.raw)
    assert d == "", d
    assert stats_dict(st) == est
    assert est["rows_read"] == rows


def test_shuffled_10m_rows_bitexact(ref, tmp_path):
    """SURVEY §8d's adversarial variant at scale: 20k journeys (~10M rows) of the bench generator
    with every row shuffled across 8 shards, so the full (rank, ts) sort path runs."""
    import numpy as np
    import paper_2305_07454_b200 as cvlg
    blob, offs, rows = cvlg.synth_day(seed=2, journeys=20_000, shards=4, mean_duration=500.0)
    body = []
    for i in range(4):
        lines = blob[offs[i]:offs[i + 1]].tobytes().split(b"\n")
        body.extend(l for l in lines[1:] if l)
    rng = np.random.default_rng(7)
    order = rng.permutation(len(body))
    body = [body[k] for k in order]
    shards = [HEADER + b"\n" + b"\n".join(body[i::8]) + b"\n" for i in range(8)]
    paths = write_shards(tmp_path, shards)
    ep, er, est, _ = ref.run_pipeline(paths, spec_default(), None, n_partitions=32, n_threads=16)
    st = cvlg.PipelineStats()
    lat = cvlg.run_pipeline(paths, spec_default(), stats=st)
    d = diff_lattice(ep, er, lat.planes, lat.raw)
    assert d == "", d
    assert stats_dict(st) == est
    assert est["rows_read"] == rows


@pytest.mark.parametrize("mode", ["windows", "no-windows", "bin-groups"])
def test_fine_grid_reopened_bins(ref, tmp_path, monkeypatch, mode):
    """c5's fine lattice (1-minute bins, 0.01-degree cells) over days that revisit the same time
    bins: reloads of flushed window blocks, spilled windows, the same with the window path off,
    and the (journey, bin) group fold (groups spanning several days)."""
    import paper_2305_07454_b200 as cvlg
    monkeypatch.setenv("CVLG_FOLD_WINDOWS", "0" if mode == "no-windows" else "1")
    monkeypatch.setenv("CVLG_FOLD_GROUPS", "1" if mode == "bin-groups" else "0")
    fine = cvlg.GridSpec(lat_step=0.01, lon_step=0.01, min_step=1)
    for cells, days in ((6, 4), (16, 3)):
        paths = write_shards(tmp_path / f"c{cells}", commuter_days(300, days, cells, seed=cells))
        assert_parity(ref, paths, fine)
        assert_parity(ref, shuffle_rows(paths, tmp_path / f"s{cells}", 3, seed=5), fine)


def test_c5_shape_fine_grid_7_days_bitexact(ref, tmp_path):
    """configs[4]'s shape on one GPU: 7 consecutive days of the bench generator with the same
    journey ids (10k journeys, ~35M rows) on the 1-minute / 0.01-degree lattice."""
    import datetime
    import os
    import paper_2305_07454_b200 as cvlg
    blobs = []
    for k in range(7):
        d = (datetime.date(2021, 5, 9) + datetime.timedelta(days=k)).isoformat()
        blob, offs, _ = cvlg.synth_day(seed=1 + k, journeys=10_000, shards=2, mean_duration=500.0,
                                       day=d)
        blobs += [blob[offs[i]:offs[i + 1]].tobytes() for i in range(2)]
    paths = write_shards(tmp_path, blobs)
    fine = cvlg.GridSpec(lat_step=0.01, lon_step=0.01, min_step=1)
    threads = max(1, min(16, os.cpu_count() or 1))
    ep, er, est, _ = ref.run_pipeline(paths, fine, None, n_partitions=2 * threads,
                                      n_threads=threads)
    st = cvlg.PipelineStats()
    lat = cvlg.run_pipeline(paths, fine, stats=st)
    d = diff_lattice(ep, er, lat.planes, lat.raw)
    assert d == "", d
    assert stats_dict(st) == est


def test_randomized_differential(ref, day_cache, tmp_path):
    """48 seeded random cases against cvl::run_pipeline: generator settings (journeys, shard count,
    sample period < 1 for duplicates, mean duration, bbox partly off-grid), a random valid grid
    (steps, minute bins, direction sectors and offset), filter rules, optional row shuffling
    across shards and optional multi-day manifests."""
    import paper_2305_07454_b200 as cvlg
    rng = random.Random(2305)
    steps = [0.5, 0.25, 0.1, 0.05, 0.02, 0.013]
    mins = [1, 2, 5, 15, 30, 60, 1440]
    dxns = [(90, 0.0), (90, 45.0), (120, -30.0), (180, 10.0), (360, 0.0)]
    for case in range(48):
        seed = 100 + case
        journeys = rng.choice([5, 20, 60])
        period = rng.choice([1.0, 1.0, 0.5])
        bbox = rng.choice([None, (35.0, 41.0, -96.5, -88.5)])
        paths, _ = day_cache(seed=seed, journeys=journeys, shards=rng.choice([1, 3, 8]),
                             sample_period=period, mean_duration=rng.choice([60.0, 200.0]),
                             bbox=bbox)
        if rng.random() < 0.3:
            more, _ = day_cache(seed=seed + 1000, journeys=journeys, shards=2, day="2021-05-10")
            paths = paths + more
        if rng.random() < 0.3:
            paths = shuffle_rows(paths, tmp_path / f"s{case}", rng.choice([2, 5]), seed=case)
        while True:  # a random grid of at most 40M cells (the reference's frames are dense)
            step = rng.choice(steps)
            dxn, off = rng.choice(dxns)
            spec = cvlg.GridSpec(lat_step=step,
                                 lon_step=rng.choice(steps) if rng.random() < 0.3 else step,
                                 min_step=rng.choice(mins), dxn_step=dxn, dxn_offset=off)
            t, d, r, c = spec.dims()
            if t * d * r * c <= 40_000_000:
                break
        rules = cvlg.FilterRules(require_in_grid=True, speed_ceiling=rng.choice([250.0, 100.0]))
        assert_parity(ref, paths, spec, rules)


def test_daily_bins_fine_cells_spill_retry(ref, tmp_path):
    """One time bin per day (min_step = 1440) on 0.01-degree cells over 3 days: every journey is a
    single time-bin window holding ~150 cells, so the fold's window tables spill into the
    (cell, journey) hash table, which overflows its first size and re-runs larger."""
    import os
    import paper_2305_07454_b200 as cvlg
    blobs = []
    for k in range(3):
        blob, offs, _ = cvlg.synth_day(seed=50 + k, journeys=12_000, shards=2, mean_duration=500.0,
                                       day="2021-05-%02d" % (9 + k))
        blobs += [blob[offs[i]:offs[i + 1]].tobytes() for i in range(2)]
    paths = write_shards(tmp_path, blobs)
    spec = cvlg.GridSpec(lat_step=0.01, lon_step=0.01, min_step=1440)
    threads = max(1, min(16, os.cpu_count() or 1))
    ep, er, est, _ = ref.run_pipeline(paths, spec, None, n_partitions=2 * threads, n_threads=threads)
    st = cvlg.PipelineStats()
    lat = cvlg.run_pipeline(paths, spec, stats=st)
    d = diff_lattice(ep, er, lat.planes, lat.raw)
    assert d == "", d
    assert stats_dict(st) == est


@pytest.mark.parametrize("groups", ["1", "0"])
def test_few_long_journeys_bin_groups(ref, tmp_path, monkeypatch, groups):
    """Few, long journeys (the fold's lanes would each carry one journey): the (journey, time bin)
    group fold against the reference, default and fine grids, and the journey fold it replaces."""
    import paper_2305_07454_b200 as cvlg
    monkeypatch.setenv("CVLG_FOLD_GROUPS", groups)
    blob, offs, _ = cvlg.synth_day(seed=9, journeys=150, shards=3, mean_duration=9000.0)
    paths = write_shards(tmp_path, [blob[offs[i]:offs[i + 1]].tobytes() for i in range(3)])
    assert_parity(ref, paths, cvlg.GridSpec())
    assert_parity(ref, paths, cvlg.GridSpec(lat_step=0.01, lon_step=0.01, min_step=1))
