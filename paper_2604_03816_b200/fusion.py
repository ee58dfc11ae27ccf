"""DAG gate fusion, mirrored from the reference pass (``aqsim.dag``).

The B200 engine consumes the *output* of this pass:
fused ops are CUSTOM gates on an ascending qubit union, and they are lowered
by the native planner (``csrc/planner.cpp``) into multi-gate tile passes.

The pass is re-implemented here (not imported) so the engine has no runtime
dependency on the reference package; its semantics follow Alg. 2 of the paper
as shipped in ``pkg/src/aqsim/dag.py``:

* wire DAG: an edge u->v iff u is the latest earlier gate on a qubit of v
  (ref dag.py:77-90);
* Kahn topological order with program order as the tie-break (ref dag.py:51-66);
* v merges into predecessor u iff the qubit union fits ``max_fuse_width``,
  u is v's immediate predecessor on every shared wire, and (width >= 3 case)
  no other predecessor of v is reachable from u (ref dag.py:123-138);
* the merged op is CUSTOM on ``sorted(union)`` with matrix
  ``expand(U_v) @ expand(U_u)`` computed in complex128 (ref dag.py:141-174);
* passes repeat until a full sweep merges nothing (ref dag.py:177-217).

Given the same input, the output gate list (order, targets, matrices) equals
the reference's; ``tests/test_fusion.py`` pins that against the golden
fixtures that ``tests/golden/make_golden.py`` made with ``aqsim.dag.fuse``.
"""
from __future__ import annotations

import heapq
import time
from dataclasses import dataclass

from .circuit import Circuit, GateKind, GateOp, effective_unitary, expand_unitary, require_valid


@dataclass
class FusionReport:
    """Same fields as ``aqsim.dag.FusionReport`` (ref dag.py:98-105)."""

    original_gate_count: int
    fused_gate_count: int
    original_depth: int
    fused_depth: int
    reduction_percent: float
    fusion_pass_time: float


class _WireDag:
    """Per-qubit linked wires over gate nodes; node id = original gate index."""

    def __init__(self, circuit):
        require_valid(circuit)
        self.ops: dict[int, object] = {}
        self.rank: dict[int, int] = {}          # program-order key (never changes)
        self.prev: dict[int, dict[int, int]] = {}
        self.next: dict[int, dict[int, int]] = {}
        tail: dict[int, int] = {}
        for i, op in enumerate(circuit.gates):
            self.ops[i] = op
            self.rank[i] = i
            self.prev[i] = {}
            self.next[i] = {}
            for q in op.targets:
                if q in tail:
                    self.prev[i][q] = tail[q]
                    self.next[tail[q]][q] = i
                tail[q] = i

    def qubits(self, v: int) -> frozenset:
        return frozenset(self.ops[v].targets)

    def preds(self, v: int) -> set:
        return set(self.prev[v].values())

    def succs(self, v: int) -> set:
        return set(self.next[v].values())

    def topo(self) -> list[int]:
        indeg = {v: len(self.preds(v)) for v in self.ops}
        heap = [(self.rank[v], v) for v, d in indeg.items() if d == 0]
        heapq.heapify(heap)
        out = []
        while heap:
            _, v = heapq.heappop(heap)
            out.append(v)
            for w in self.succs(v):
                indeg[w] -= 1
                if indeg[w] == 0:
                    heapq.heappush(heap, (self.rank[w], w))
        if len(out) != len(self.ops):
            raise RuntimeError("dependency graph contains a cycle")
        return out

    def depth(self) -> int:
        level: dict[int, int] = {}
        for v in self.topo():
            level[v] = 1 + max((level[u] for u in self.preds(v)), default=0)
        return max(level.values(), default=0)

    def reaches(self, src: int, goals: set, blocked: int) -> bool:
        seen = {src, blocked}
        todo = [src]
        while todo:
            x = todo.pop()
            for y in self.succs(x):
                if y in goals:
                    return True
                if y not in seen:
                    seen.add(y)
                    todo.append(y)
        return False

    def can_absorb(self, u: int, v: int, width: int) -> bool:
        qu, qv = self.qubits(u), self.qubits(v)
        if len(qu | qv) > width:
            return False
        for w in qu & qv:
            if self.prev[v].get(w) != u:
                return False
        if (qu - qv) and (qv - qu):
            others = self.preds(v) - {u}
            if others and self.reaches(u, others, blocked=v):
                return False
        return True

    def absorb(self, u: int, v: int) -> None:
        """Replace u by the product 'v after u' on the sorted qubit union."""
        qu, qv = self.qubits(u), self.qubits(v)
        union = sorted(qu | qv)
        slot = {q: j for j, q in enumerate(union)}
        wide_u = expand_unitary(effective_unitary(self.ops[u]),
                                [slot[t] for t in self.ops[u].targets], len(union))
        wide_v = expand_unitary(effective_unitary(self.ops[v]),
                                [slot[t] for t in self.ops[v].targets], len(union))
        merged = GateOp(GateKind.CUSTOM, tuple(union), (), wide_v @ wide_u)
        new_prev: dict[int, int] = {}
        new_next: dict[int, int] = {}
        for q in union:
            src_prev = self.prev[u] if q in qu else self.prev[v]
            src_next = self.next[v] if q in qv else self.next[u]
            if q in src_prev:
                new_prev[q] = src_prev[q]
            if q in src_next:
                new_next[q] = src_next[q]
        self.ops[u] = merged
        self.prev[u] = new_prev
        self.next[u] = new_next
        for q, p in new_prev.items():
            self.next[p][q] = u
        for q, s in new_next.items():
            self.prev[s][q] = u
        for table in (self.ops, self.rank, self.prev, self.next):
            del table[v]


def depth(circuit) -> int:
    """Longest dependency path in gates (ref dag.py:93-95)."""
    return _WireDag(circuit).depth()


def fuse(circuit, max_fuse_width: int = 2):
    """Fusion pass; returns ``(fused_circuit, FusionReport)`` (ref dag.py:177-217)."""
    if max_fuse_width not in (1, 2, 3):
        raise ValueError(f"max_fuse_width must be 1, 2, or 3, got {max_fuse_width}")
    depth0 = depth(circuit)
    t0 = time.perf_counter()
    dag = _WireDag(circuit)
    progress = True
    while progress:
        progress = False
        for v in dag.topo():
            if v not in dag.ops:
                continue
            for u in sorted(dag.preds(v), key=lambda x: (dag.rank[x], x)):
                if dag.can_absorb(u, v, max_fuse_width):
                    dag.absorb(u, v)
                    progress = True
                    break
    fused = Circuit(circuit.num_qubits, [dag.ops[v] for v in dag.topo()],
                    getattr(circuit, "name", ""))
    elapsed = time.perf_counter() - t0
    depth1 = depth(fused)
    reduction = 100.0 * (1.0 - depth1 / depth0) if depth0 > 0 else 0.0
    return fused, FusionReport(len(circuit.gates), len(fused.gates), depth0, depth1,
                               reduction, elapsed)
