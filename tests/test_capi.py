"""CPU tests (no GPU): the C-ABI library loads, exports every symbol include/cvlg.h declares, and
its host-side logic (grid validation, error codes, container writer, synthetic generator)
matches the reference. No kernel is launched here."""
from __future__ import annotations

import ctypes
import hashlib
import json
import re
import tempfile
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"


def declared_symbols() -> list[str]:
    text = (ROOT / "include" / "cvlg.h").read_text()
    return sorted(set(re.findall(r"\b(cvlg_[a-z_]+)\s*\(", text)))


def test_library_exports_header_symbols():
    import paper_2305_07454_b200.cvlg as c
    lib = ctypes.CDLL(str(c.LIB_PATH))
    syms = declared_symbols()
    assert len(syms) >= 14
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(c.EXPORTED_SYMBOLS) <= set(syms)


def test_library_is_sm100a():
    import paper_2305_07454_b200.cvlg as c
    import shutil
    import subprocess
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([cuobjdump, "--list-elf", str(c.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out, out


def test_grid_dims_and_validation():
    import paper_2305_07454_b200 as cvlg
    assert cvlg.GridSpec().dims() == (288, 4, 46, 67)
    assert cvlg.GridSpec(lat_min=36.0, lat_max=36.1, lon_min=-93.0, lon_max=-92.8, lat_step=0.01,
                         lon_step=0.01).dims() == (288, 4, 10, 20)
    assert cvlg.GridSpec(lat_step=10.0, lon_step=10.0).dims()[2:] == (1, 1)
    for bad in [dict(lat_max=36.0), dict(min_step=7), dict(dxn_step=100), dict(lat_step=0.0),
                dict(dxn_offset=float("inf")), dict(lon_min=-89.1)]:
        with pytest.raises(cvlg.CvlError) as e:
            cvlg.GridSpec(**bad).dims()
        assert e.value.code == "BadGrid"
    with pytest.raises(cvlg.CvlError) as e:
        cvlg.GridSpec(dxn_step=45).dims()  # 8 direction planes: BatchFrame holds 4
    assert e.value.code == "Unsupported"


def test_grid_dims_match_golden():
    import paper_2305_07454_b200 as cvlg
    for e in json.loads((GOLDEN / "grid_kat.json").read_text()):
        g = cvlg.GridSpec(**e["grid"])
        assert g.dims()[2:] == (e["rows"], e["cols"])


@pytest.mark.parametrize("case", ["synth_small", "malformed", "table1"])
def test_container_writer_matches_reference_bytes(case, tmp_path):
    import paper_2305_07454_b200 as cvlg
    d = GOLDEN / "days" / case
    meta = json.loads((d / "expected.json").read_text())
    planes = np.load(d / "expected.npz")["planes"]
    spec = cvlg.GridSpec(**meta["grid"])
    p = tmp_path / "x.cvl1"
    n = cvlg.write_container(planes, spec, 18756, p)
    assert n == p.stat().st_size
    assert hashlib.sha256(p.read_bytes()).hexdigest() == meta["container_sha256_day18756"]


def test_container_rejects_non_finite(tmp_path):
    import paper_2305_07454_b200 as cvlg
    spec = cvlg.GridSpec(lat_step=10.0, lon_step=10.0)
    t, _, r, c = spec.dims()
    planes = np.zeros((t, 8, r, c), dtype=np.uint32)
    planes[3, 1, 0, 0] = 0x7FC00000  # NaN speed
    with pytest.raises(cvlg.CvlError) as e:
        cvlg.write_container(planes, spec, 0, tmp_path / "x.cvl1")
    assert e.value.code == "NonFiniteValue"


def test_synth_matches_reference_generator(ref, tmp_path):
    """The threaded bench generator is byte-identical to the reference generate_day."""
    import paper_2305_07454_b200 as cvlg
    for kw in [dict(seed=3, journeys=30, shards=4, mean_duration=120.0),
               dict(seed=9, journeys=17, shards=5, sample_period=0.5, mean_duration=40.0,
                    day="1999-12-31")]:
        blob, offs, rows = cvlg.synth_day(**kw)
        d = tmp_path / str(kw["seed"])
        total = ref.generate_day(d, **kw)
        assert total == rows
        for s in range(kw["shards"]):
            assert (d / f"shard_{s:04d}.csv").read_bytes() == blob[offs[s]:offs[s + 1]].tobytes()


def test_synth_golden_sha():
    """Generator pinned without the reference: golden synth_small shards."""
    import paper_2305_07454_b200 as cvlg
    d = GOLDEN / "days" / "synth_small"
    blob, offs, _ = cvlg.synth_day(seed=1, journeys=24, shards=3, mean_duration=150.0)
    for s in range(3):
        assert (d / f"shard_{s:04d}.csv").read_bytes() == blob[offs[s]:offs[s + 1]].tobytes()


def test_no_cpu_fallback_in_product():
    """The product package never imports the oracle (the checker)."""
    pkg = ROOT / "paper_2305_07454_b200"
    for f in pkg.rglob("*.py"):
        assert "oracle" not in f.read_text().replace("oracle/", ""), f
