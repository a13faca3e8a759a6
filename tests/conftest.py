import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"
CASES = ROOT / "cases"
FIXTURES = sorted(p.stem for p in GOLDEN.glob("fx_*.ptc"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: large cases (c1..c5) when their caches exist")


def golden_path(name):
    return GOLDEN / f"{name}.ptc"


def case_path(name):
    return CASES / f"{name}.ptc"


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True
