import gzip
import json
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))
os.environ.setdefault("TESSEL_BUDGET_SECS", "1e9")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def load_search(name):
    return json.loads((GOLDEN / f"search_{name}.json").read_text())


def load_probes(name):
    with gzip.open(GOLDEN / f"probes_{name}.json.gz", "rt") as f:
        return json.load(f)["probes"]


def probe_names():
    return sorted(p.name[len("probes_"):-len(".json.gz")] for p in GOLDEN.glob("probes_*.json.gz"))


def search_names():
    return sorted(p.name[len("search_"):-len(".json")] for p in GOLDEN.glob("search_*.json")
                  if p.name != "search_random.json")


@pytest.fixture(scope="session")
def gpu():
    """Skip unless a CUDA device and the in-tree library are present."""
    from paper_2311_15269_b200 import _native

    _native.build()
    if _native.device_count() < 1:
        pytest.skip("no CUDA device")
    return _native
