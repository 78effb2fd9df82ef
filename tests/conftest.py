import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


def _has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    for item in items:
        if "gpu" in item.keywords and not HAS_GPU:
            item.add_marker(pytest.mark.skip(reason="no CUDA device"))


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Ref
    if not Ref.available():
        pytest.skip("oracle/_ref not built")
    return Ref()


@pytest.fixture(scope="session")
def day_cache(tmp_path_factory):
    """Synthetic days from the reference generator (synth.cpp:145), cached per session."""
    from oracle.oracle import Ref
    cache = {}
    root = tmp_path_factory.mktemp("days")

    def get(seed=1, journeys=100, shards=8, sample_period=1.0, mean_duration=300.0,
            day="2021-05-09", bbox=None):
        key = (seed, journeys, shards, sample_period, mean_duration, day, bbox)
        if key not in cache:
            d = root / ("d%d" % len(cache))
            rows = Ref().generate_day(d, seed=seed, journeys=journeys, shards=shards,
                                      sample_period=sample_period, mean_duration=mean_duration,
                                      day=day, bbox=bbox)
            paths = sorted(str(p) for p in d.glob("*.csv"))
            cache[key] = (paths, rows)
        return cache[key]

    return get
