"""Benchmark circuit families used by the bench and the parity tests.

* ``layered_circuit`` -- the seeded H/RX/RZ + CNOT-brick + RZ generator that
  BASELINE.json's configs call "random layered circuit" (defined in SURVEY.md
  section 8(d); it is not in the reference package).  Seed 0 gives depth 42
  that fuses to 14 at every width.
* ``qft_circuit`` -- the reference's QFT with each controlled phase decomposed
  into RZ/CNOT/RZ/CNOT/RZ (ref ``pkg/src/aqsim/generators.py:37-57``).
* ``random_su2_circuit`` -- the paper's Table-2 workload, Haar U3 on uniform
  targets (ref ``generators.py:60-77``).
"""
from __future__ import annotations

import math

import numpy as np

from .circuit import Circuit, GateKind, GateOp


def layered_circuit(num_qubits: int, layers: int = 14, seed: int = 0,
                    kinds=None) -> Circuit:
    """per layer, H|RX|RZ on every qubit, CNOT brick at offset
    ``L % 2``, then RZ on every qubit; angles uniform in [0, 2pi)."""
    ops = kinds or (GateKind.H, GateKind.RX, GateKind.RZ)
    rng = np.random.default_rng(seed)
    gates: list[GateOp] = []
    for layer in range(layers):
        for q in range(num_qubits):
            kind = ops[int(rng.integers(0, 3))]
            if kind is GateKind.H:
                gates.append(GateOp(kind, (q,)))
            else:
                gates.append(GateOp(kind, (q,), (rng.uniform(0, 2 * math.pi),)))
        for q in range(layer % 2, num_qubits - 1, 2):
            gates.append(GateOp(GateKind.CNOT, (q, q + 1)))
        for q in range(num_qubits):
            gates.append(GateOp(GateKind.RZ, (q,), (rng.uniform(0, 2 * math.pi),)))
    return Circuit(num_qubits, gates, name=f"layered-{num_qubits}")


def _cphase(control: int, target: int, theta: float) -> list[GateOp]:
    half = theta / 2
    return [GateOp(GateKind.RZ, (control,), (half,)),
            GateOp(GateKind.CNOT, (control, target)),
            GateOp(GateKind.RZ, (target,), (-half,)),
            GateOp(GateKind.CNOT, (control, target)),
            GateOp(GateKind.RZ, (target,), (half,))]


def qft_circuit(num_qubits: int) -> Circuit:
    if num_qubits < 1:
        raise ValueError("num_qubits must be >= 1")
    gates: list[GateOp] = []
    for t in range(num_qubits):
        gates.append(GateOp(GateKind.H, (t,)))
        for c in range(t + 1, num_qubits):
            gates.extend(_cphase(c, t, math.pi / (1 << (c - t))))
    return Circuit(num_qubits, gates, name=f"qft-{num_qubits}")


def random_su2_circuit(num_qubits: int, num_gates: int, seed: int) -> Circuit:
    if num_qubits < 1:
        raise ValueError("num_qubits must be >= 1")
    rng = np.random.default_rng(seed)
    gates = []
    for _ in range(num_gates):
        q = int(rng.integers(0, num_qubits))
        theta = 2.0 * math.asin(math.sqrt(rng.random()))
        phi = rng.uniform(0.0, 2.0 * math.pi)
        lam = rng.uniform(0.0, 2.0 * math.pi)
        gates.append(GateOp(GateKind.U3, (q,), (theta, phi, lam)))
    return Circuit(num_qubits, gates, name=f"random-{num_qubits}")


def ghz_circuit(num_qubits: int) -> Circuit:
    if num_qubits < 2:
        raise ValueError("a GHZ circuit needs at least 2 qubits")
    gates = [GateOp(GateKind.H, (0,))]
    gates += [GateOp(GateKind.CNOT, (q, q + 1)) for q in range(num_qubits - 1)]
    return Circuit(num_qubits, gates, name=f"ghz-{num_qubits}")
