import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs under gpurun / the round-end GPU tier)")
    config.addinivalue_line("markers", "slow: larger parity cases")


@pytest.fixture(scope="session")
def golden():
    import json
    manifest = json.loads((GOLDEN / "manifest.json").read_text())
    images = {p.stem: p.read_bytes() for p in GOLDEN.glob("*.bin")}
    return manifest, images


@pytest.fixture(scope="session")
def eng():
    from paper_2008_10596_b200 import engine
    engine.lib()
    return engine
