"""Multi-GPU data plane: journey-hash routing of data lines and the
time-slab combine.

CPU (no GPU): the manifest split (host code of the library) covers every data byte exactly once
at line boundaries; the exchange layout of distributed.py (stream_layout / virtual_shards) run
over gloo with world_size 2 on streams built by the routing restatement (tests/route_oracle.py,
hashing with the reference's own journey_hash) gives owners whose virtual shards, run through the
UNMODIFIED reference cvl::run_pipeline as one manifest, reproduce the original lattice and stats
bit for bit — i.e. routing keeps every row, keeps each journey's rows in provenance order and
never splits a journey.

GPU (one device): the routing kernels' streams equal the restatement's byte for byte, and the
whole multi-GPU pipeline — one host thread driving N "GPUs" (contexts on the same device), and
two processes exchanging over torch.distributed — equals the reference bit for bit.
"""
from __future__ import annotations

import os
import socket
from pathlib import Path

import numpy as np
import pytest

from helpers import HEADER, commuter_days, diff_lattice, malformed_contents, shuffle_rows, \
    stats_dict, write_shards
import route_oracle


def _ranked(paths):
    return sorted(str(p) for p in paths)


def _id_cols(ref, paths_ranked):
    cols = []
    for p in paths_ranked:
        hdr, _ = route_oracle.header_of(p)
        line = hdr[:-1]
        if line.endswith(b"\r"):
            line = line[:-1]
        c = ref.parse_header(line) if Path(p).stat().st_size else None
        cols.append(c[0] if c else -1)
    return cols


def _datasets(tmp_path, day_cache):
    sets = {}
    sets["synth"] = day_cache(seed=41, journeys=160, shards=8)[0]
    sets["malformed"] = write_shards(tmp_path / "bad", malformed_contents(11))
    sets["shuffled"] = shuffle_rows(day_cache(seed=42, journeys=80, shards=4)[0], tmp_path / "shuf", 5, 3)
    sets["dups"] = day_cache(seed=43, journeys=60, shards=3, sample_period=0.5)[0]
    return sets


# ---- CPU ------------------------------------------------------------------------------------------
@pytest.mark.parametrize("n_parts", [1, 2, 3, 5, 8])
def test_split_manifest_covers_every_data_byte(tmp_path, day_cache, n_parts):
    import paper_2305_07454_b200 as cvlg
    for name, paths in _datasets(tmp_path / str(n_parts), day_cache).items():
        ranked = _ranked(paths)
        got = []
        for part in range(n_parts):
            got += cvlg.cvlg.split_manifest(ranked, n_parts, part)
        # pieces in provenance order, contiguous, exactly the data bytes of the good shards
        expect = []
        for r, p in enumerate(ranked):
            data = Path(p).read_bytes()
            if not data:
                continue
            hdr, first = route_oracle.header_of(p)
            line = hdr[:-1].rstrip(b"\r")
            if not line.lower().replace(b" ", b"").startswith(b"journeyid") and b"journey" not in line.lower():
                continue  # the BadHeader shard
            if first < len(data):
                expect.append((r, first, len(data) - first))
        merged = []
        for f, o, ln in got:
            data = Path(ranked[f]).read_bytes()
            assert o == 0 or data[o - 1:o] == b"\n", (name, f, o)  # starts at a line start
            assert o + ln == len(data) or data[o + ln - 1:o + ln] == b"\n", (name, f, o, ln)
            if merged and merged[-1][0] == f and merged[-1][1] + merged[-1][2] == o:
                merged[-1] = (f, merged[-1][1], merged[-1][2] + ln)
            else:
                merged.append((f, o, ln))
        assert merged == expect, name


def test_stream_layout_and_virtual_shards():
    from paper_2305_07454_b200.distributed import slab_rows, stream_layout, virtual_shards
    lens = [[5, 7], [11, 13]]
    base, recv = stream_layout(lens)
    assert recv == [16, 20] and base == [[0, 0], [5, 7]]
    plans = [([[0, 2], [0, 3]], [5, 7]), ([[0], [0]], [11, 13])]
    assert virtual_shards(plans, 0) == [0, 2, 5, 16]
    assert virtual_shards(plans, 1) == [0, 3, 7, 20]
    import paper_2305_07454_b200 as cvlg
    for T in (1, 24, 288, 1440):
        for n in (1, 2, 3, 5, 8, 16):
            rows = [slab_rows(T, n, r) for r in range(n)]
            assert rows[0][0] == 0 and rows[-1][1] == T
            assert all(rows[i][1] == rows[i + 1][0] for i in range(n - 1))
            assert all(cvlg.cvlg.slab_rows(T, n, r) == rows[r] for r in range(n))
            for t in range(T):
                o = t * n // T
                assert rows[o][0] <= t < rows[o][1]


def _gloo_worker(rank, world, port, paths, out_dir, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2305_07454_b200 as cvlg
        from paper_2305_07454_b200.distributed import all_gather_obj, all_to_all_bytes, virtual_shards
        from oracle.oracle import Ref
        ref = Ref()
        ranked = _ranked(paths)
        cols = _id_cols(ref, ranked)
        pieces = cvlg.cvlg.split_manifest(ranked, world, rank)
        streams, vs = route_oracle.streams(ranked, pieces, cols, world, ref.journey_hash)
        lens = [len(s) for s in streams]
        plans = all_gather_obj((vs, lens))
        send = torch.frombuffer(bytearray(b"".join(streams) or b"\0"), dtype=torch.uint8)[: sum(lens)]
        recv = all_to_all_bytes(send, lens, [p[1][rank] for p in plans]).numpy().tobytes()
        offs = virtual_shards(plans, rank)
        owned = set()
        for i in range(len(offs) - 1):
            blob = recv[offs[i]:offs[i + 1]]
            (Path(out_dir) / f"o{rank}_{i:06d}.csv").write_bytes(blob)
            lines = blob.split(b"\n")
            cols = ref.parse_header(lines[0].rstrip(b"\r"))
            for raw in lines[1:]:
                if raw and raw != b"\r":
                    f = raw.rstrip(b"\r").split(b",")
                    owned.add(f[cols[0]].strip(b" \t\r") if cols[0] < len(f) else b"")
        q.put((rank, sorted(owned), None))
    except Exception as e:  # pragma: no cover
        q.put((rank, None, repr(e)))
    finally:
        dist.destroy_process_group()


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("name", ["synth", "malformed", "shuffled", "dups"])
def test_gloo_routing_preserves_the_reference_result(ref, tmp_path, day_cache, name):
    import torch.multiprocessing as mp
    import paper_2305_07454_b200 as cvlg
    paths = _datasets(tmp_path / "in", day_cache)[name]
    out = tmp_path / "routed"
    out.mkdir()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, paths, str(out), q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(err is None for *_, err in res), res
    # journeys are disjoint across owners
    assert not (set(res[0][1]) & set(res[1][1]))
    spec = cvlg.GridSpec(lat_step=0.25, lon_step=0.25)
    ep, er, est, _ = ref.run_pipeline(paths, spec, n_partitions=3)
    routed = sorted(str(p) for p in out.glob("*.csv"))
    gp, gr, gst, _ = ref.run_pipeline(routed, spec, n_partitions=3)
    assert diff_lattice(ep, er, gp, gr) == ""
    bad = est["rejected"].pop("BadHeader", 0)
    gst["rejected"].pop("BadHeader", None)
    assert gst == est, (gst, est)
    assert bad in (0, 1)


# ---- GPU ------------------------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("n_parts", [2, 3, 8])
def test_route_kernels_match_restatement(ref, tmp_path, day_cache, n_parts):
    import ctypes
    import torch
    import paper_2305_07454_b200 as cvlg
    lib = cvlg.cvlg.lib()
    for name, paths in _datasets(tmp_path / str(n_parts), day_cache).items():
        ranked = _ranked(paths)
        cols = _id_cols(ref, ranked)
        arr = (ctypes.c_char_p * len(ranked))(*[p.encode() for p in ranked])
        ctx = cvlg.Context()
        for part in range(n_parts):
            pieces = cvlg.cvlg.split_manifest(ranked, n_parts, part)
            exp, exp_vs = route_oracle.streams(ranked, pieces, cols, n_parts, ref.journey_hash)
            npc, bad = ctypes.c_uint64(), ctypes.c_uint64()
            cvlg.cvlg._check(lib.cvlg_route_stage(ctx.handle, arr, len(ranked), n_parts, part, 2,
                                                  ctypes.byref(npc), ctypes.byref(bad)))
            assert npc.value == len(pieces)
            bufs = []
            for o in range(n_parts):
                vs = (ctypes.c_uint64 * max(len(pieces), 1))()
                ln = ctypes.c_uint64()
                cvlg.cvlg._check(lib.cvlg_route_plan(ctx.handle, o, vs, ctypes.byref(ln)))
                assert ln.value == len(exp[o]), (name, part, o)
                assert [vs[i] for i in range(len(pieces))] == exp_vs[o], (name, part, o)
                bufs.append(torch.zeros(ln.value + 8, dtype=torch.uint8, device="cuda"))
            dst = (ctypes.c_void_p * n_parts)(*[b.data_ptr() for b in bufs])
            cvlg.cvlg._check(lib.cvlg_route_scatter(ctx.handle, dst, None))
            for o in range(n_parts):
                got = bufs[o][: len(exp[o])].cpu().numpy().tobytes()
                assert got == exp[o], (name, part, o)
        ctx.close()


@pytest.mark.gpu
@pytest.mark.parametrize("n_gpus", [1, 2, 3, 8])
def test_multi_gpu_pipeline_matches_reference(ref, tmp_path, day_cache, n_gpus):
    """One host thread, n_gpus contexts on device 0: routed, aggregated per owner, combined by
    time slab — the reference's lattice and stats bit for bit."""
    import paper_2305_07454_b200 as cvlg
    sets = _datasets(tmp_path / "in", day_cache)
    sets["multiday_fine"] = write_shards(tmp_path / "md", commuter_days(120, 3, 6, seed=5))
    m = cvlg.MultiGPU([0] * n_gpus)
    for name, paths in sets.items():
        spec = (cvlg.GridSpec(lat_step=0.01, lon_step=0.01, min_step=1) if name == "multiday_fine"
                else cvlg.GridSpec())
        ep, er, est, _ = ref.run_pipeline(paths, spec, n_partitions=3, n_threads=1)
        st = cvlg.PipelineStats()
        lat = m.run_pipeline(paths, spec, stats=st)
        d = diff_lattice(ep, er, lat.planes, lat.raw)
        assert d == "", (name, d)
        assert stats_dict(st) == est, name
        one = cvlg.run_pipeline(paths, spec)
        assert np.array_equal(one.planes, lat.planes) and np.array_equal(one.raw, lat.raw)
    m.close()


@pytest.mark.gpu
@pytest.mark.parametrize("n_gpus", [1, 2, 5])
def test_multi_gpu_long_ids(ref, tmp_path, n_gpus):
    """Ids longer than the 15-byte inline key: journeys keyed by global ranks (host merge of
    every GPU's sorted ids), including ids that share a 15-byte prefix."""
    import random
    import paper_2305_07454_b200 as cvlg
    rng = random.Random(3)
    ids = ([b"vehicle-%012d" % i for i in range(30)] + [b"x" * n for n in range(1, 25)]
           + [b"prefix-shared-%d-tail" % i for i in range(12)] + [b"j%06d" % i for i in range(20)])
    rows = []
    for k in range(5000):
        j = rng.choice(ids)
        rows.append(b"%s,2021-05-09 %02d:%02d:%02d,%.6f,%.6f,65101,%.2f,%.2f" % (
            j, rng.randrange(24), rng.randrange(60), rng.randrange(60), 36.2 + rng.random() * 0.5,
            -95.5 + rng.random() * 0.5, rng.uniform(0, 120), rng.uniform(0, 360)))
    paths = write_shards(tmp_path, [HEADER + b"\n" + b"\n".join(rows[i::3]) + b"\n" for i in range(3)])
    spec = cvlg.GridSpec(lat_step=0.25, lon_step=0.25)
    ep, er, est, _ = ref.run_pipeline(paths, spec)
    m = cvlg.MultiGPU([0] * n_gpus)
    st = cvlg.PipelineStats()
    lat = m.run_pipeline(paths, spec, stats=st)
    assert diff_lattice(ep, er, lat.planes, lat.raw) == ""
    assert stats_dict(st) == est
    m.close()


def _torchrun_worker(rank, world, port, paths, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2305_07454_b200 as cvlg
        from paper_2305_07454_b200.distributed import FileShardedPipeline
        spec = cvlg.GridSpec()
        runner = FileShardedPipeline(paths, spec, ctx=cvlg.Context(0), threads=2)
        st = cvlg.PipelineStats()
        lat = runner.run_files(stats=st)
        T, _, R, C = spec.dims()
        d_planes = torch.empty((T, 8, R, C), dtype=torch.int32, device="cuda")
        d_raw = torch.empty((T, 4, R, C), dtype=torch.int32, device="cuda")
        runner.run_resident(d_planes, d_raw)
        same = (np.array_equal(d_planes.cpu().numpy().view(np.uint32), lat.planes)
                and np.array_equal(d_raw.cpu().numpy().view(np.uint32), lat.raw))
        q.put((rank, lat.planes, lat.raw, stats_dict(st), same, None))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, None, None, None, False, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_process_per_rank_pipeline_matches_reference(ref, tmp_path, day_cache):
    """distributed.FileShardedPipeline with two processes (gloo moves the bytes; both ranks on
    device 0): every rank ends with the reference's lattice and stats."""
    import torch.multiprocessing as mp
    import paper_2305_07454_b200 as cvlg
    paths = _datasets(tmp_path / "in", day_cache)["malformed"] + \
        [str(p) for p in day_cache(seed=44, journeys=50, shards=2)[0]]
    ep, er, est, _ = ref.run_pipeline(paths, cvlg.GridSpec(), n_partitions=2)
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_torchrun_worker, args=(r, world, port, paths, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, planes, raw, st, same, err in res:
        assert err is None, err
        assert diff_lattice(ep, er, planes, raw) == ""
        assert st == est
        assert same
