import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))  # test infrastructure: the parity checker

GOLDEN = ROOT / "tests" / "golden" / "golden.json"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    # Build the native libraries and the oracle when absent (nvcc cross-compiles
    # without a GPU); the product path has no fallback if this fails.
    from paper_2201_10956_b200 import build as b
    lib = ROOT / "paper_2201_10956_b200" / "libepi3cu.so"
    olib = ROOT / "oracle" / "_build" / "libepi3_oracle.so"
    if not lib.exists() or not olib.exists() or not b.LIB_CPP.exists():
        b.build_all()


@pytest.fixture(scope="session")
def golden():
    return json.loads(GOLDEN.read_text())


@pytest.fixture(scope="session")
def golden_cases(golden):
    return {c["name"]: c for c in golden["cases"]}
