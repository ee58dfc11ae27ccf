"""Drop-in boundary on CPU: importing the package registers "b200" into the
reference's registry (opt-in, ref engines.py:267-292) with the accelerator flag
that makes ``aqsim.selector.select`` skip it when no GPU is present
(ref selector.py:155-157)."""
from __future__ import annotations

import os
import sys

import pytest

REF = "/root/reference/pkg/src"


_CHECK = r"""
import sys
sys.path.insert(0, {ref!r})
sys.path.insert(0, {root!r})
import aqsim
from aqsim import selector
import paper_2604_03816_b200 as P
names = {{e.name for e in aqsim.registered_engines()}}
assert {{"reference", "parallel", "b200"}} <= names, names
eng = aqsim.get_engine("b200")
assert isinstance(eng, aqsim.Engine)
assert eng.id.requires_accelerator
assert issubclass(P.AllocationError, aqsim.AllocationError)
if not eng.is_available():
    choice, profiles = selector.select(aqsim.ghz_circuit(4), aqsim.registered_engines())
    assert choice.name in {{"reference", "parallel"}}
    assert all(p.engine.name != "b200" for p in profiles)
print("ok")
"""


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference package only in the build container")
def test_registration_and_selector_tolerance():
    # fresh interpreter: the package binds to aqsim's Engine at import time
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, "-c", _CHECK.format(ref=REF, root=root)],
                         capture_output=True, text=True, timeout=300)
    assert res.returncode == 0 and "ok" in res.stdout, res.stderr


def test_own_registry_has_b200():
    import paper_2604_03816_b200 as P
    assert "b200" in {e.name for e in P.registered_engines()}
    with pytest.raises(KeyError):
        P.get_engine("nope")
    with pytest.raises(ValueError):
        P.register_engine(P.get_engine("b200"))
