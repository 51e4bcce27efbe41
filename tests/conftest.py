"""Shared test plumbing.

Markers: `gpu` = needs a CUDA device (parity tests through the C ABI / pybind module). The CPU
suite (-m "not gpu") covers the oracle against the golden vectors, the host-side API and the
C-ABI library's exported symbols.
"""
import hashlib
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests of the sm_100a path")
    config.addinivalue_line("markers", "slow: long-running (full-size configurations)")


def golden(name):
    with open(os.path.join(GOLDEN, name + ".json")) as f:
        meta = json.load(f)
    npz = os.path.join(GOLDEN, name + ".npz")
    arrays = dict(np.load(npz)) if os.path.exists(npz) else {}
    return meta, arrays


def golden_names(prefix=""):
    return sorted(f[:-5] for f in os.listdir(GOLDEN) if f.endswith(".json") and f.startswith(prefix))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="session")
def f2m():
    import paper_2011_08170_b200 as mod
    return mod


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle as o
    return o


@pytest.fixture(scope="session")
def ref():
    """The UNMODIFIED reference module (oracle/_ref/f2m), when it has been built."""
    path = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.exists(os.path.join(path, "f2m", "__init__.py")):
        pytest.skip("oracle/_ref not built (make -C oracle ref)")
    if path not in sys.path:
        sys.path.insert(0, path)
    import f2m as reference
    return reference
