"""The C-ABI library loads on a CPU host and exports every symbol of include/svb200.h."""
from __future__ import annotations

import ctypes
import os
import re

from conftest import ROOT
from paper_2604_03816_b200 import _native


def declared_symbols() -> set[str]:
    text = open(os.path.join(ROOT, "include", "svb200.h")).read()
    return set(re.findall(r"\b(svb_[a-z0-9_]+)\s*\(", text))


def test_header_and_binding_agree():
    assert declared_symbols() == set(_native.EXPORTS)


def test_library_exports_all_symbols():
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert _native.lib().svb_abi_version() == _native.ABI_VERSION


def test_errors_map_to_python_exceptions():
    import numpy as np
    import pytest
    ks = np.array([1], dtype=np.int32)
    tg = np.zeros((1, 8), dtype=np.int32)
    tg[0, 0] = 5
    mats = np.eye(2, dtype=np.complex128).reshape(-1).view(np.float64)
    with pytest.raises(ValueError, match="out of range"):
        _native.NativePlan(3, _native.SVB_C128, ks, tg, mats)
    assert "out of range" in _native.lib().svb_last_error().decode()
