"""Engine API mirrored from the reference (``aqsim.engines``), host side.

The reference's plugin boundary is the ``Engine`` class plus a module-level
registry (ref ``pkg/src/aqsim/engines.py:110-187, 267-302``).  This module
provides the same names for environments without the reference package; when
``aqsim`` *is* importable, the B200 engine subclasses the reference's own
``Engine`` and registers into the reference's registry instead
(``paper_2604_03816_b200.b200``), so ``aqsim.run_circuit("b200", ...)`` works.

Nothing here computes amplitudes: the only engine this package ships is the
CUDA one.  ``state_fidelity`` promotes to complex128 on the host exactly as
ref ``engines.py:340-346`` does; the engine also offers device-side
reductions (``B200Engine.fidelity``).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .circuit import Precision, as_precision

try:  # the reference package, when present, is the base we plug into
    import aqsim.engines as _ref_engines  # type: ignore
except Exception:  # pragma: no cover - depends on the environment
    _ref_engines = None


if _ref_engines is not None:
    class AllocationError(_ref_engines.AllocationError):
        """Device allocation refused (also an ``aqsim.AllocationError``)."""
else:
    class AllocationError(Exception):
        """State allocation refused (ref engines.py:31-43)."""

        def __init__(self, requested_bytes: int, capacity_bytes: int | None):
            self.requested_bytes = requested_bytes
            self.capacity_bytes = capacity_bytes
            super().__init__(f"requested {requested_bytes} bytes does not fit within engine "
                             f"capacity {capacity_bytes}")


@dataclass
class SampleResult:
    """Measurement counts keyed by bitstring, qubit 0 rightmost (ref engines.py:52-57)."""

    counts: dict
    shots: int


@dataclass(frozen=True)
class EngineId:
    name: str
    requires_accelerator: bool = False


@dataclass
class StateVector:
    """Host state (ref circuit.py:187-205): 2^n amplitudes, little-endian."""

    num_qubits: int
    precision: Precision
    amplitudes: np.ndarray

    def norm_squared(self) -> float:
        return float(np.sum(np.abs(self.amplitudes.astype(np.complex128)) ** 2))

    def probabilities(self) -> np.ndarray:
        return np.abs(self.amplitudes.astype(np.complex128)) ** 2


class Engine:
    """Interface of ref engines.py:110-187 (used only when aqsim is absent)."""

    def __init__(self, name: str, *, requires_accelerator: bool = False,
                 capacity_bytes: int | None = None):
        self.id = EngineId(name, requires_accelerator)
        self.capacity_bytes = capacity_bytes
        self.live_states = 0

    @property
    def name(self) -> str:
        return self.id.name

    def is_available(self) -> bool:
        return True

    def init_state(self, num_qubits: int, precision):
        raise NotImplementedError

    def adopt(self, num_qubits: int, precision, amplitudes):
        raise NotImplementedError

    def release(self, state) -> None:
        del state
        self.live_states -= 1

    def apply_gate(self, state, op):
        raise NotImplementedError

    def synchronize(self) -> None:
        """Barrier for engines with asynchronous kernels."""

    def run_circuit(self, circuit, precision=Precision.DOUBLE, checkpoint=None):
        state = self.init_state(circuit.num_qubits, precision)
        for i, op in enumerate(circuit.gates):
            if checkpoint is not None:
                checkpoint(state, i)
            self.apply_gate(state, op)
        self.synchronize()
        return state


EngineBase = _ref_engines.Engine if _ref_engines is not None else Engine

_REGISTRY: dict[str, object] = {}


def register_engine(engine) -> None:
    if engine.name in _REGISTRY:
        raise ValueError(f"engine {engine.name!r} already registered")
    _REGISTRY[engine.name] = engine


def get_engine(name: str):
    try:
        return _REGISTRY[name]
    except KeyError:
        raise KeyError(f"unknown engine {name!r}; registered: {sorted(_REGISTRY)}") from None


def available_engines() -> list:
    return [e.id for e in _REGISTRY.values() if e.is_available()]


def registered_engines() -> list:
    return list(_REGISTRY.values())


def run_circuit(engine, circuit, precision=Precision.DOUBLE, checkpoint=None):
    """Run on an engine given by instance, id or registered name (ref engines.py:295-302)."""
    if isinstance(engine, str):
        engine = get_engine(engine)
    elif hasattr(engine, "name") and not hasattr(engine, "run_circuit"):
        engine = get_engine(engine.name)
    return engine.run_circuit(circuit, precision, checkpoint=checkpoint)


def state_fidelity(a, b) -> float:
    """|<a|b>|^2 with both promoted to complex128 (ref engines.py:340-346)."""
    if a.num_qubits != b.num_qubits:
        raise ValueError(f"qubit counts differ: {a.num_qubits} vs {b.num_qubits}")
    ov = np.vdot(np.asarray(a.amplitudes).astype(np.complex128),
                 np.asarray(b.amplitudes).astype(np.complex128))
    return float(abs(ov) ** 2)


__all__ = ["AllocationError", "Engine", "EngineBase", "EngineId", "StateVector",
           "register_engine", "get_engine", "available_engines", "registered_engines",
           "run_circuit", "state_fidelity", "as_precision"]
