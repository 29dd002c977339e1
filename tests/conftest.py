"""Shared fixtures.  `-m "not gpu"` runs on CPU only (oracle vs golden vectors,
host logic, C-ABI symbol checks, gloo multi-process); `-m gpu` tests are the
parity tests proper and call the CUDA path through the C ABI."""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")
    config.addinivalue_line("markers", "slow: long-running (large-size properties)")


def _ensure_built():
    import __graft_entry__
    __graft_entry__.build()


@pytest.fixture(scope="session")
def built():
    _ensure_built()
    return True


@pytest.fixture(scope="session")
def port(built):
    import oracle
    return oracle.Oracle("port")


@pytest.fixture(scope="session")
def ref(built):
    import oracle
    if not oracle.available("ref"):
        pytest.skip("reference build (oracle/_ref) not present")
    return oracle.Oracle("ref")


@pytest.fixture(scope="session")
def ctx(built):
    from paper_2005_10680_b200 import _native as nat
    if nat.device_count() < 1:
        pytest.fail("GPU test scheduled but no CUDA device is visible")
    return nat.Context(0)


def load_golden(name: str):
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def golden_names():
    import json
    return json.loads((GOLDEN / "manifest.json").read_text())["cases"]


def bits(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, np.float64)).view(np.uint64)


def bits_equal(x, y) -> bool:
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    return x.shape == y.shape and np.array_equal(bits(x), bits(y))
