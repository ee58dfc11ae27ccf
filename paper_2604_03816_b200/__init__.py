"""B200-native state-vector engine for the gate-application path of arXiv 2604.03816.

Importing the package registers the ``"b200"`` engine: into this package's
registry always, and into the reference package's registry (``aqsim``) when
that package is importable -- opt-in registration, so the reference's own
test-suite, which pins the default engine set (ref pkg/tests/test_engines.py:15),
is unaffected unless this package is imported.
"""
from __future__ import annotations

from .circuit import (Circuit, GateKind, GateOp, Precision, effective_unitary, expand_unitary,
                      gate_matrix, validate)
from .engines import (AllocationError, EngineId, StateVector, available_engines, get_engine,
                      register_engine, registered_engines, run_circuit, state_fidelity)
from .fusion import FusionReport, depth, fuse
from .precision import PrecisionDecision, select_precision
from .b200 import B200Engine, CircuitPlan, DeviceStateVector, plan_options

__version__ = "0.1.0"

ENGINE_NAME = "b200"


def _register() -> None:
    eng = B200Engine(ENGINE_NAME, devices="all")  # shards over the box's GPUs when a state does not fit one
    if ENGINE_NAME not in {e.name for e in registered_engines()}:
        register_engine(eng)
    try:
        import aqsim.engines as ref  # type: ignore
    except Exception:
        return
    if ENGINE_NAME not in {e.name for e in ref.registered_engines()}:
        ref.register_engine(eng)


_register()

__all__ = ["Circuit", "GateKind", "GateOp", "Precision", "effective_unitary", "expand_unitary",
           "gate_matrix", "validate", "AllocationError", "EngineId", "StateVector",
           "available_engines", "get_engine", "register_engine", "registered_engines",
           "run_circuit", "state_fidelity", "FusionReport", "depth", "fuse",
           "PrecisionDecision", "select_precision", "B200Engine", "CircuitPlan",
           "DeviceStateVector", "plan_options"]
