"""Test configuration: the `gpu` marker selects tests that need a B200.

The driver runs `pytest -m "not gpu"` in the CPU build container and
`pytest -m gpu` on a GPU box. GPU tests call the CUDA path through the
C-ABI and check it against the CPU oracle (oracle/) and the golden vectors
produced by the reference itself (tests/golden/).
"""
import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a kernels")


@pytest.fixture(scope="session")
def golden():
    meta = json.loads((GOLDEN / "reference_vectors.json").read_text())
    arrays = dict(np.load(GOLDEN / "reference_vectors.npz"))
    return meta, arrays


def unpack(packed_u8, n):
    return np.unpackbits(np.asarray(packed_u8, np.uint8), bitorder="little")[:n]
