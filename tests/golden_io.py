"""(De)serialisation of circuits + states for the golden fixtures in tests/golden/.

A circuit is stored as parallel arrays (kind names, -1-padded targets,
0-padded params, 0-padded 8x8 matrices for CUSTOM ops) so the fixtures are
plain ``.npz`` files that need neither the reference package nor pickle.
"""
from __future__ import annotations

import numpy as np

from paper_2604_03816_b200.circuit import Circuit, GateKind, GateOp


def encode(prefix: str, circuit, out: dict) -> None:
    g = len(circuit.gates)
    kinds = np.array([op.kind.value for op in circuit.gates] or [""], dtype="U8")[:g]
    tg = -np.ones((g, 3), dtype=np.int64)
    pr = np.zeros((g, 3), dtype=np.float64)
    mats = np.zeros((g, 8, 8), dtype=np.complex128)
    for i, op in enumerate(circuit.gates):
        tg[i, :len(op.targets)] = op.targets
        pr[i, :len(op.params)] = op.params
        if op.matrix is not None:
            d = op.matrix.shape[0]
            mats[i, :d, :d] = op.matrix
    out[prefix + "n"] = np.int64(circuit.num_qubits)
    out[prefix + "kinds"] = kinds
    out[prefix + "targets"] = tg
    out[prefix + "params"] = pr
    out[prefix + "mats"] = mats


def decode(prefix: str, z) -> Circuit:
    n = int(z[prefix + "n"])
    gates = []
    for i, kind in enumerate(z[prefix + "kinds"]):
        kind = GateKind(str(kind))
        tg = tuple(int(t) for t in z[prefix + "targets"][i] if t >= 0)
        if kind is GateKind.CUSTOM:
            d = 1 << len(tg)
            gates.append(GateOp(kind, tg, (), z[prefix + "mats"][i, :d, :d]))
        else:
            gates.append(GateOp(kind, tg, tuple(z[prefix + "params"][i, :kind.param_count])))
    return Circuit(n, gates)
