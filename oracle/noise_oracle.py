"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY (see sv_oracle.py's header).

Restatement of the reference's density-matrix noise arm,
``pkg/src/aqsim/noise.py:61-102`` (``evolve_noisy``): rho = |0><0|; per gate
rho <- U rho U^dagger with U the full-space unitary (``expand_unitary``,
ref ``circuit.py:275-295``), then for every qubit the gate touches, in target
order, the depolarizing channel of ``noise.py:52-58``:
rho <- (1 - p) rho + (p / 3) (X rho X + Y rho Y + Z rho Z).
Pinned against fixtures the reference itself produced
(``tests/golden/make_noise_golden.py`` -> ``noise_golden.npz``).
"""
from __future__ import annotations

import numpy as np

from .sv_oracle import gate_unitary

_X = np.array([[0, 1], [1, 0]], dtype=complex)
_Y = np.array([[0, -1j], [1j, 0]], dtype=complex)
_Z = np.array([[1, 0], [0, -1]], dtype=complex)


def expand(u: np.ndarray, targets, n: int) -> np.ndarray:
    """Full-space matrix of u on `targets` (local bit j <-> targets[j]),
    entry placement as ref circuit.py:275-295."""
    k = len(targets)
    dim = 1 << n
    out = np.zeros((dim, dim), dtype=complex)
    rest = [q for q in range(n) if q not in targets]
    for other in range(1 << (n - k)):
        base = 0
        for j, q in enumerate(rest):
            base |= ((other >> j) & 1) << q
        idx = [base | sum(((a >> j) & 1) << t for j, t in enumerate(targets)) for a in range(1 << k)]
        out[np.ix_(idx, idx)] = u
    return out


def evolve_noisy(circuit, p: float) -> np.ndarray:
    n = circuit.num_qubits
    dim = 1 << n
    rho = np.zeros((dim, dim), dtype=complex)
    rho[0, 0] = 1.0
    paulis = {}
    for op in circuit.gates:
        u = expand(gate_unitary(op), list(op.targets), n)
        rho = u @ rho @ u.conj().T
        if p > 0.0:
            for q in op.targets:
                if q not in paulis:
                    paulis[q] = tuple(expand(m, [q], n) for m in (_X, _Y, _Z))
                x, y, z = paulis[q]
                rho = (1.0 - p) * rho + (p / 3.0) * (x @ rho @ x + y @ rho @ y + z @ rho @ z)
    return rho
