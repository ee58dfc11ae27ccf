"""Shared test configuration.

* registers the ``gpu`` marker: ``-m gpu`` tests need a B200 and the built
  CUDA library; ``-m "not gpu"`` tests run on any CPU host;
* puts the repo root and ``tests/`` on sys.path so tests import the package,
  the oracle (test infrastructure) and ``golden_io``.
"""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"
# the unmodified reference package installed by the driver's one offline
# install (`pip install --target baseline/_ref /root/reference/pkg`); it
# travels to the GPU box, so the drop-in tests (aqsim.run_circuit("b200"),
# selector profiling) run there too.  Appended, never shadowing the repo.
REFERENCE_INSTALL = os.path.join(ROOT, "baseline", "_ref")
if os.path.isdir(os.path.join(REFERENCE_INSTALL, "aqsim")) and REFERENCE_INSTALL not in sys.path:
    sys.path.append(REFERENCE_INSTALL)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 and the built libsvb200.so")


@pytest.fixture(scope="session")
def golden_random():
    return np.load(os.path.join(GOLDEN, "random_circuits.npz"))


@pytest.fixture(scope="session")
def golden_fused():
    return np.load(os.path.join(GOLDEN, "fused_circuits.npz"))


def has_cuda() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False
