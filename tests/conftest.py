"""pytest configuration: the `gpu` marker and shared fixtures.

`-m "not gpu"` tests run on any host (planner, minimax, oracle vs golden vectors, C-ABI
symbol/loading checks, gloo multi-process sharding logic).  `-m gpu` tests need a B200
and exercise the sm_100a kernels through the C ABI; they fail (not skip) when no device
is present, so a silent fallback can never pass them.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run with -m gpu")


@pytest.fixture(scope="session")
def pft():
    import paper_2008_12559_b200 as m
    m.lib()  # fail loudly if the library is missing
    return m


@pytest.fixture(scope="session")
def oracle():
    import oracle as o
    o.lib()
    return o


@pytest.fixture
def rng():
    return np.random.default_rng(20260419)
