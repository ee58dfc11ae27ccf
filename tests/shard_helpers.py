"""CPU stand-ins for the sharded engine's device backend (TEST INFRASTRUCTURE).

``OracleShardBackend`` applies a shard's local segment with the oracle's
numpy kernels on a CPU torch tensor, so the scheduler, the exchange protocol
(torch.distributed point-to-point over gloo) and the layout bookkeeping of
``paper_2604_03816_b200.sharded`` can be tested without a GPU.
"""
from __future__ import annotations

import numpy as np
import torch

from oracle import sv_oracle as orc
from paper_2604_03816_b200.circuit import as_precision
from paper_2604_03816_b200.sharded import LocalStep, SwapStep, block_peer, localize, own_block, schedule, unpermute

_DT = {"single": torch.complex64, "double": torch.complex128}


class _Shard:
    def __init__(self, n_local, precision):
        self.num_qubits = n_local
        self.precision = as_precision(precision)
        self.tensor = torch.zeros(1 << n_local, dtype=_DT[self.precision.value])


class OracleShardBackend:
    def alloc(self, n_local, precision):
        return _Shard(n_local, precision)

    def fill(self, state, index_of_one):
        state.tensor.zero_()
        if index_of_one >= 0:
            state.tensor[index_of_one] = 1

    def plan(self, n_local, precision, gates):
        return list(gates)

    def run(self, state, plan):
        a = state.tensor.numpy()
        for op in plan:
            orc.apply_gate(a, state.num_qubits, op)

    def tensor(self, state):
        return state.tensor

    def norm2(self, state):
        a = state.tensor.numpy().astype(np.complex128)
        return float(np.vdot(a, a).real)

    def synchronize(self):
        pass


def simulate(circuit, world: int, precision="double") -> np.ndarray:
    """Single-process 'virtual ranks' execution of a schedule."""
    sched = schedule(circuit, world)
    nl = sched.n_local
    shards = [orc.init_state(nl, precision) if r == 0 else
              np.zeros(1 << nl, dtype=orc.dtype_of(precision)) for r in range(world)]
    for st in sched.steps:
        if isinstance(st, LocalStep):
            for r, a in enumerate(shards):
                for op in localize(st.gates, nl, r):
                    orc.apply_gate(a, nl, op)
        else:
            blk = 1 << (nl - st.m)
            old = [a.copy() for a in shards]
            for r in range(world):
                for w in range(1 << st.m):
                    if w == own_block(r, st):
                        continue
                    p = block_peer(r, st, w)
                    src = own_block(r, st)
                    shards[r][w * blk:(w + 1) * blk] = old[p][src * blk:(src + 1) * blk]
    return unpermute(np.concatenate(shards), sched.n, sched.final_layout), sched
