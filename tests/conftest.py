import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built sm_100a library")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    cases = json.loads((GOLDEN / "cases.json").read_text())
    vec = np.load(GOLDEN / "vectors.npz")
    front = json.loads((GOLDEN / "frontend.json").read_text())
    return {"cases": cases["cases"], "c1": cases["c1"], "underflow": cases["underflow"],
            "vec": vec, "front": front}
