"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference package's state-vector path, used as
the parity checker for the B200 engine.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it; the product package never does.

What it restates (all citations into /root/reference):

* gate matrices: ``pkg/src/aqsim/circuit.py:91-152`` (fixed table, RX/RY/RZ,
  U3), CUSTOM returns the stored matrix (``circuit.py:208-214``);
* ``init_state``: zeros + amp[0] = 1 (``engines.py:130-140``);
* ``apply_gate``: range check, matrix rounded to the state dtype *before* use
  (``engines.py:152-162``, the c64 rounding at line 157);
* 1-qubit kernel: strided pair views + butterfly, written back through the
  views (``engines.py:62-80``);
* k-qubit kernel: index arrays with zero bits inserted at the sorted targets,
  gather, row-by-row accumulation in column order, scatter
  (``engines.py:83-105``);
* ``state_fidelity``: |vdot|^2 after promotion to complex128
  (``engines.py:340-346``);
* an independent full-matrix oracle (permutation + kron) for n <= 6, the
  reference tests' anchor (``pkg/tests/conftest.py:27-54``).

The arithmetic is expressed with the same numpy operations in the same order
as the reference, so on the same numpy build the results are bit-identical
to ``aqsim``'s ReferenceEngine -- ``tests/test_oracle.py`` pins this against
golden vectors produced by the reference itself (``tests/golden/make_golden.py``).
"""
from __future__ import annotations

import math

import numpy as np

_R2 = 1.0 / math.sqrt(2.0)


def _name(kind) -> str:
    return kind.value if hasattr(kind, "value") else str(kind)


def gate_unitary(op) -> np.ndarray:
    """complex128 unitary of an op (ref circuit.py:91-152, 208-214)."""
    name = _name(op.kind)
    p = tuple(float(x) for x in op.params)
    if name == "CUSTOM":
        return np.asarray(op.matrix, dtype=complex)
    table = {
        "I": [[1, 0], [0, 1]],
        "X": [[0, 1], [1, 0]],
        "Y": [[0, -1j], [1j, 0]],
        "Z": [[1, 0], [0, -1]],
        "S": [[1, 0], [0, 1j]],
        "T": [[1, 0], [0, np.exp(1j * math.pi / 4)]],
        "CNOT": [[1, 0, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0], [0, 1, 0, 0]],
        "CZ": np.diag([1, 1, 1, -1]),
        "SWAP": [[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]],
    }
    if name == "H":
        return np.array([[1, 1], [1, -1]], dtype=complex) * _R2
    if name in table:
        return np.array(table[name], dtype=complex)
    if name == "TOFFOLI":
        m = np.eye(8, dtype=complex)
        m[[3, 7]] = m[[7, 3]]
        return m
    if name == "RX":
        c, s = math.cos(p[0] / 2), math.sin(p[0] / 2)
        return np.array([[c, -1j * s], [-1j * s, c]], dtype=complex)
    if name == "RY":
        c, s = math.cos(p[0] / 2), math.sin(p[0] / 2)
        return np.array([[c, -s], [s, c]], dtype=complex)
    if name == "RZ":
        return np.array([[np.exp(-1j * p[0] / 2), 0], [0, np.exp(1j * p[0] / 2)]],
                        dtype=complex)
    if name == "U3":
        th, ph, la = p
        c, s = math.cos(th / 2), math.sin(th / 2)
        return np.array([[c, -np.exp(1j * la) * s],
                         [np.exp(1j * ph) * s, np.exp(1j * (ph + la)) * c]], dtype=complex)
    raise ValueError(f"oracle: unknown gate kind {name}")


def dtype_of(precision) -> np.dtype:
    v = getattr(precision, "value", precision)
    return np.dtype(np.complex64 if v == "single" else np.complex128)


def init_state(num_qubits: int, precision) -> np.ndarray:
    """|0...0> (ref engines.py:130-140)."""
    if num_qubits < 1:
        raise ValueError("num_qubits must be >= 1")
    amps = np.zeros(1 << num_qubits, dtype=dtype_of(precision))
    amps[0] = 1.0
    return amps


def _pair_halves(amps: np.ndarray, t: int):
    # ref engines.py:70-80
    if t == 0:
        v = amps.reshape(-1, 2)
        return v[:, 0], v[:, 1]
    v = amps.reshape(-1, 2, 1 << t)
    return v[:, 0, :], v[:, 1, :]


def _butterfly(a: np.ndarray, b: np.ndarray, u: np.ndarray) -> None:
    # ref engines.py:62-67 -- same expression order
    lo = u[0, 0] * a + u[0, 1] * b
    hi = u[1, 0] * a + u[1, 1] * b
    a[:] = lo
    b[:] = hi


def _group_offsets(n: int, targets) -> list[np.ndarray]:
    # ref engines.py:94-105
    q = len(targets)
    base = np.arange(1 << (n - q), dtype=np.intp)
    for t in sorted(targets):
        base = ((base >> t) << (t + 1)) | (base & ((1 << t) - 1))
    return [base + sum(1 << targets[b] for b in range(q) if (j >> b) & 1)
            for j in range(1 << q)]


def _group_apply(amps: np.ndarray, u: np.ndarray, idx) -> None:
    # ref engines.py:83-91 -- gather, accumulate in column order, scatter
    cols = [amps[ix] for ix in idx]
    for i in range(len(idx)):
        acc = u[i, 0] * cols[0]
        for j in range(1, len(idx)):
            acc += u[i, j] * cols[j]
        amps[idx[i]] = acc


def apply_gate(amps: np.ndarray, num_qubits: int, op) -> np.ndarray:
    """In-place gate application (ref engines.py:152-162, 196-203)."""
    tg = tuple(int(t) for t in op.targets)
    if any(not 0 <= t < num_qubits for t in tg):
        raise ValueError(f"target out of range for {num_qubits} qubits: {tg}")
    u = gate_unitary(op).astype(amps.dtype)
    if len(tg) == 1:
        a, b = _pair_halves(amps, tg[0])
        _butterfly(a, b, u)
    else:
        _group_apply(amps, u, _group_offsets(num_qubits, tg))
    return amps


def _group_offsets_range(n: int, targets, g0: int, g1: int) -> list[np.ndarray]:
    # _group_offsets restricted to groups [g0, g1) (ref engines.py:94-105)
    q = len(targets)
    base = np.arange(g0, g1, dtype=np.intp)
    for t in sorted(targets):
        base = ((base >> t) << (t + 1)) | (base & ((1 << t) - 1))
    return [base + sum(1 << targets[b] for b in range(q) if (j >> b) & 1)
            for j in range(1 << q)]


def apply_gate_parallel(amps: np.ndarray, num_qubits: int, op, pool, workers: int) -> np.ndarray:
    """The reference's chunked data-parallel kernels (ref ParallelEngine,
    engines.py:206-262) generalised from 2 to `workers` chunks: contiguous
    slices of the pair views / of the group range, each run by the reference
    kernel on a pool thread (numpy releases the GIL).  Element-wise the same
    arithmetic as apply_gate, hence bit-identical results (as
    ref test_engines.py:105-117 pins for the 2-chunk engine)."""
    tg = tuple(int(t) for t in op.targets)
    if any(not 0 <= t < num_qubits for t in tg):
        raise ValueError(f"target out of range for {num_qubits} qubits: {tg}")
    u = gate_unitary(op).astype(amps.dtype)
    if workers < 2 or amps.size < (1 << 16):
        return apply_gate(amps, num_qubits, op)
    if len(tg) == 1:
        a, b = _pair_halves(amps, tg[0])
        ax = 0 if (a.ndim == 1 or a.shape[0] >= workers) else 1
        n = a.shape[ax]
        cuts = [n * w // workers for w in range(workers + 1)]
        sl = [(slice(cuts[w], cuts[w + 1]),) if ax == 0 else (slice(None), slice(cuts[w], cuts[w + 1]))
              for w in range(workers)]
        futs = [pool.submit(_butterfly, a[x], b[x], u) for x in sl]
    else:
        groups = amps.size >> len(tg)
        cuts = [groups * w // workers for w in range(workers + 1)]

        def chunk(g0, g1):
            _group_apply(amps, u, _group_offsets_range(num_qubits, tg, g0, g1))
        futs = [pool.submit(chunk, cuts[w], cuts[w + 1]) for w in range(workers)]
    for f in futs:
        f.result()
    return amps


def apply_matrix(amps: np.ndarray, num_qubits: int, targets, u: np.ndarray) -> np.ndarray:
    """Apply an explicit 2^k x 2^k matrix with the reference kernels."""
    class _Op:  # minimal CUSTOM op
        kind = "CUSTOM"
        params = ()
    op = _Op()
    op.targets = tuple(targets)
    op.matrix = u
    return apply_gate(amps, num_qubits, op)


def run_circuit(circuit, precision="double") -> np.ndarray:
    """init_state then every gate in order (ref engines.py:174-187)."""
    amps = init_state(circuit.num_qubits, precision)
    for op in circuit.gates:
        apply_gate(amps, circuit.num_qubits, op)
    return amps


def state_fidelity(a: np.ndarray, b: np.ndarray) -> float:
    """Unnormalised |<a|b>|^2 in complex128 (ref engines.py:340-346)."""
    if a.shape != b.shape:
        raise ValueError(f"qubit counts differ: {a.shape} vs {b.shape}")
    return float(abs(np.vdot(a.astype(np.complex128), b.astype(np.complex128))) ** 2)


def normalised_fidelity(a: np.ndarray, b: np.ndarray) -> float:
    """|<a|b>|^2 / (<a|a><b|b>) in FP64 -- the c64 parity metric."""
    a = a.astype(np.complex128)
    b = b.astype(np.complex128)
    num = abs(np.vdot(a, b)) ** 2
    den = float(np.vdot(a, a).real) * float(np.vdot(b, b).real)
    return float(num / den)


# --- independent full-matrix oracle (ref pkg/tests/conftest.py:27-54) --------

def kron_embed(u: np.ndarray, targets, n: int) -> np.ndarray:
    q = len(targets)
    order = list(targets) + [t for t in range(n) if t not in targets]
    dim = 1 << n
    perm = np.zeros((dim, dim))
    for k in range(dim):
        kp = 0
        for pos, old in enumerate(order):
            kp |= ((k >> old) & 1) << pos
        perm[kp, k] = 1.0
    return perm.T @ np.kron(np.eye(1 << (n - q)), u) @ perm


def kron_state(circuit) -> np.ndarray:
    """Column 0 of the explicit product of embedded gate matrices (n <= ~8)."""
    n = circuit.num_qubits
    total = np.eye(1 << n, dtype=complex)
    for op in circuit.gates:
        total = kron_embed(gate_unitary(op), op.targets, n) @ total
    return total[:, 0].copy()
