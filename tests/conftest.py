"""Shared test setup.

* ``-m gpu`` tests need a B200 (the CUDA engine); everything else runs on CPU.
* The CPU oracle (oracle/, test infrastructure) is built on first use.
* Golden fixtures come from tests/golden/make_golden.py (the reference run in
  the build container); /root/reference is never read here.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built engine")
    config.addinivalue_line("markers", "slow: longer-running test")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as fh:
        meta = json.load(fh)
    arrays = dict(np.load(os.path.join(GOLDEN, "golden.npz")))
    return meta, arrays


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O

    O.build()
    return O


def bits(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64)).view(np.uint64)


def same_float(a: float, b: float) -> bool:
    """Bit-identical doubles (NaN == NaN)."""
    return np.float64(a).view(np.uint64) == np.float64(b).view(np.uint64) or (
        np.isnan(a) and np.isnan(b))


def servers_from_rows(rows, mod):
    return tuple(mod.ServerSpec(r[0], int(r[1]), float(r[2]), float(r[3])) for r in rows)
