"""Multi-GPU combine logic.

CPU (gloo, world_size 2): the slab partition + all-to-all exchange (distributed.all_to_all_bytes)
+ per-rank fold + slab gather reproduces a single-process fold of the union of tuples
(the fold here is a numpy restatement of the reference finalize, aggregate.cpp:161-204 — test
code only). GPU (1 device): the C-ABI building blocks (partial -> export -> finalize) over two
journey-hash shards give the lattice of the single-shard pipeline bit for bit.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def np_finalize(cols: np.ndarray, T, D, R, C):
    """cols: (n, 5) int64 = cell, key0, key1, sum bits, count -> planes [T,8,R,C], raw."""
    planes = np.zeros((T, 8, R, C), dtype=np.uint32)
    raw = np.zeros((T, 4, R, C), dtype=np.uint32)
    if len(cols) == 0:
        return planes, raw
    u = cols.view(np.uint64)
    order = np.lexsort((u[:, 2], u[:, 1], u[:, 0]))
    c = cols[order]
    sums = c[:, 3].copy().view(np.float64)
    RC = R * C
    i = 0
    while i < len(c):
        j = i
        s = 0.0
        n = 0
        while j < len(c) and c[j, 0] == c[i, 0]:
            s += float(sums[j])
            n += int(c[j, 4])
            j += 1
        g = int(c[i, 0])
        t, d, rc = g // (D * RC), (g // RC) % D, g % RC
        planes[t, d].reshape(-1)[rc] = np.float32(s / n).view(np.uint32)
        planes[t, 4 + d].reshape(-1)[rc] = j - i
        raw[t, d].reshape(-1)[rc] = n
        i = j
    return planes, raw


def make_tuples(rank: int, T, D, R, C, n=400, seed=0):
    """Disjoint journeys per rank (key0 carries the rank), random cells / subtotals."""
    rng = np.random.default_rng(seed + rank)
    cell = rng.integers(0, T * D * R * C, n)
    cell[: n // 4] = rng.integers(0, 10, n // 4)  # shared hot cells across ranks
    k0 = (rng.integers(0, 50, n) << 8) | rank
    k1 = rng.integers(0, 2 ** 40, n)
    sums = rng.uniform(0, 130, n) * rng.integers(1, 40, n)
    cnt = rng.integers(1, 300, n)
    cols = np.stack([cell, k0, k1, sums.view(np.int64), cnt], axis=1).astype(np.int64)
    # (cell, journey) unique
    _, idx = np.unique(cols[:, :3], axis=0, return_index=True)
    return cols[np.sort(idx)]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2305_07454_b200.distributed import all_gather_obj, all_to_all_bytes, slab_rows
    T, D, R, C = 24, 4, 3, 5
    mine = make_tuples(rank, T, D, R, C)
    # partition by time-slab owner (owner(t) = t * world // T, route.cu tuple_owner)
    owner = (mine[:, 0] // (D * R * C)) * world // T
    order = np.argsort(owner, kind="stable")
    send = np.ascontiguousarray(mine[order])
    counts = np.bincount(owner, minlength=world).tolist()
    all_counts = all_gather_obj(counts)
    recv = all_to_all_bytes(torch.from_numpy(send.view(np.uint8).reshape(-1).copy()),
                            [c * 40 for c in counts], [c[rank] * 40 for c in all_counts])
    got = recv.numpy().view(np.int64).reshape(-1, 5)
    t0, t1 = slab_rows(T, world, rank)
    ts = got[:, 0] // (D * R * C)
    assert bool(((ts >= t0) & (ts < t1)).all())
    planes, raw = np_finalize(got, T, D, R, C)
    slabs = all_gather_obj((t0, t1, planes[t0:t1], raw[t0:t1]))
    p = np.zeros_like(planes)
    r = np.zeros_like(raw)
    for a, b, sp, sr in slabs:
        p[a:b] = sp
        r[a:b] = sr
    allc = np.concatenate([make_tuples(k, T, D, R, C) for k in range(world)])
    ep, er = np_finalize(allc, T, D, R, C)
    q.put((rank, bool(np.array_equal(p, ep)), bool(np.array_equal(r, er)), int(got.shape[0])))
    dist.destroy_process_group()


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_gloo_exchange_matches_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok_p and ok_r for _, ok_p, ok_r, _ in res), res
    assert sum(n for *_, n in res) > 0


@pytest.mark.gpu
@pytest.mark.parametrize("shards", [2, 4, 8])
@pytest.mark.parametrize("case", ["coarse", "fine_multiday"])
def test_partial_export_finalize_shards_on_one_gpu(ref, day_cache, tmp_path, case, shards):
    """Journey-hash sharding into 2/4/8 'ranks' on one GPU: union of exported tuples finalized =
    the single pipeline = the reference (fine_multiday: the fold's time-bin window reloads and
    the vacated-pair compaction run inside each rank's partial)."""
    import ctypes
    from pathlib import Path
    import paper_2305_07454_b200 as cvlg
    from paper_2305_07454_b200 import distributed as D
    from helpers import HEADER, commuter_days, write_shards

    if case == "coarse":
        paths, _ = day_cache(seed=31, journeys=150)
        spec = cvlg.GridSpec(lat_step=0.25, lon_step=0.25)
    else:
        paths = write_shards(tmp_path / "days", commuter_days(200, 3, 6, seed=2))
        spec = cvlg.GridSpec(lat_step=0.01, lon_step=0.01, min_step=1)
    rows = []
    for p in paths:
        rows += [l for l in Path(p).read_bytes().split(b"\n")[1:] if l]

    def fnv(b):
        h = 1469598103934665603
        for c in b:
            h = ((h ^ c) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
        return h

    T, Dn, R, C = spec.dims()
    tuples = []
    for rank in range(shards):
        mine = [l for l in rows if fnv(l.split(b",")[0]) % shards == rank]
        blob = HEADER + b"\n" + b"\n".join(mine) + b"\n"
        d_csv = torch.frombuffer(bytearray(blob), dtype=torch.uint8).cuda()
        ctx = cvlg.Context()
        n = ctypes.c_uint64()
        offs = (ctypes.c_uint64 * 2)(0, len(blob))
        cvlg.cvlg._check(D._lib.cvlg_partial_device(ctx.handle, ctypes.c_void_p(d_csv.data_ptr()),
                                                    offs, 1, ctypes.byref(spec._c()),
                                                    ctypes.byref(cvlg.FilterRules()._c()),
                                                    ctypes.byref(n), None, None))
        m = n.value
        cols = [torch.empty(m, dtype=torch.int64, device="cuda") for _ in range(5)]
        cvlg.cvlg._check(D._lib.cvlg_export_pairs(ctx.handle, *[ctypes.c_void_p(c.data_ptr()) for c in cols], None))
        tuples.append(torch.stack(cols, 1))
    allt = torch.cat(tuples)
    planes = torch.empty((T, 8, R, C), dtype=torch.int32, device="cuda")
    raw = torch.empty((T, 4, R, C), dtype=torch.int32, device="cuda")
    cs = [allt[:, i].contiguous() for i in range(5)]
    cvlg.cvlg._check(D._lib.cvlg_finalize_pairs(None, *[ctypes.c_void_p(c.data_ptr()) for c in cs],
                                                allt.shape[0], ctypes.byref(spec._c()),
                                                ctypes.c_void_p(planes.data_ptr()),
                                                ctypes.c_void_p(raw.data_ptr()), None))
    torch.cuda.synchronize()
    ep, er, _, _ = ref.run_pipeline(paths, spec)
    assert np.array_equal(planes.cpu().numpy().view(np.uint32), ep)
    assert np.array_equal(raw.cpu().numpy().view(np.uint32), er)
    # and the numpy restatement of the combine agrees with the device fold
    p2, r2 = np_finalize(allt.cpu().numpy(), T, Dn, R, C)
    assert np.array_equal(p2, ep) and np.array_equal(r2, er)
