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


# reference-scale cases the restated offline stage rebuilds in seconds
# (verified against tests/golden/<name>_ref.ptc), so a fresh checkout runs them
QUICK_CASES = ("c1", "c3r")


def case_path(name):
    path = CASES / f"{name}.ptc"
    if not path.exists() and name in QUICK_CASES:
        from paper_1410_5910_b200.offline.build import ensure_case
        path = ensure_case(name, out_dir=CASES)
    return path


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True
