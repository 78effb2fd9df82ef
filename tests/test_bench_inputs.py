"""CPU tests of bench.py's shared input: both arms materialise (or reuse) the SAME shard files —
the reference arm through the reference's own generate_journey (oracle/_ref, never this package),
our arm through the threaded generator — and describe the workload with the same config dict."""
from __future__ import annotations

import filecmp
import sys
from pathlib import Path
from types import SimpleNamespace

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


@pytest.fixture()
def bench(monkeypatch):
    import bench as b
    monkeypatch.setitem(b.WORKLOADS, "tiny", dict(journeys=300, shards=16, seed=3,
                                                   mean_duration=200.0, desc="tiny"))
    return b


def _args(tmp_path, **kw):
    return SimpleNamespace(workload="tiny", data_dir=str(tmp_path), threads=4, **kw)


def test_generators_write_identical_files(tmp_path, ref):
    from paper_2305_07454_b200.cvlg import synth_write_day
    a, b, c = tmp_path / "a", tmp_path / "b", tmp_path / "c"
    n1 = ref.generate_day(a, seed=3, journeys=300, shards=16, mean_duration=200.0)
    n2 = ref.generate_day_mt(b, seed=3, journeys=300, shards=16, mean_duration=200.0, threads=4)
    _, n3 = synth_write_day(c, seed=3, journeys=300, shards=16, mean_duration=200.0, threads=4)
    assert n1 == n2 == n3
    for f in sorted(a.glob("*.csv")):
        assert filecmp.cmp(f, b / f.name, shallow=False)
        assert filecmp.cmp(f, c / f.name, shallow=False)


def test_dataset_shared_between_arms(tmp_path, bench):
    args = _args(tmp_path)
    p1, m1, t1 = bench.ensure_dataset(args, bench.ref_generator(4))
    assert t1 > 0 and len(p1) == 16
    # our arm finds the reference arm's files valid and reuses them
    p2, m2, t2 = bench.ensure_dataset(args, bench.our_generator(4))
    assert t2 == 0.0 and p1 == p2 and m1 == m2
    # a damaged file invalidates the manifest: regenerated with our generator, same bytes
    Path(p1[3]).write_bytes(b"garbage")
    p3, m3, t3 = bench.ensure_dataset(args, bench.our_generator(4))
    assert t3 > 0 and m3["digest"] == m1["digest"] and m3["rows"] == m1["rows"]
    cfg = bench.config_of(args, m1, 1)
    assert cfg == bench.config_of(args, m3, 1)
    assert cfg["rows"] == m1["rows"] and cfg["csv_bytes"] == sum(s for _, s in m1["files"])


def test_groups_partition_the_manifest(bench):
    paths = [f"s{i:04d}" for i in range(128)]
    g = bench.groups_of(paths)
    assert len(g) == bench.GROUPS
    assert sorted(p for grp in g for p in grp) == paths
    assert all(len(grp) == 16 for grp in g)


def test_reference_arm_does_not_import_the_package():
    import subprocess
    code = ("import sys; sys.argv=['bench.py','--impl','reference']; import bench; "
            "assert 'paper_2305_07454_b200' not in sys.modules; "
            "from oracle.oracle import Ref; "
            "assert 'paper_2305_07454_b200' not in sys.modules; print('clean')")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True)
    assert out.returncode == 0 and "clean" in out.stdout, out.stderr
