"""Sharding behind the ``Engine`` plugin API: one process, the box's GPUs.

The reference's answer to a state that does not fit is the CPU fallback
(ref ``pkg/src/aqsim/memory.py:290-340``, reached from ``cli.py:262-263``).
The north star replaces it with sharding, and this module puts that behind
the same call: ``aqsim.run_circuit("b200", circuit)`` on 34-36 qubits gives a
``ShardedDeviceState`` instead of an ``AllocationError``.

* P = 2^g shards; shard r (on ``devices[r]``) holds the 2^(n-g) amplitudes
  whose top g *physical* index bits equal r.  The logical<->physical qubit
  permutation, the local segments, the global-qubit swaps and the diagonal
  gates restricted to a shard's global bits are those of ``sharded.py``
  (``schedule`` / ``localize``), shared with the torchrun engine.
* Local segments run as native plans on every shard's device (async, one
  stream per device); a swap exchanges blocks between shards in place with
  one kernel per device (svb_swap_blocks: loads and stores of the peer's
  half over NVLink, no staging buffer).
* Host views (``amplitudes``, ``probabilities``) and sampling first restore
  the identity layout on the device (``canonicalize``: physical SWAP gates
  on local qubits, block exchanges for global ones, a shard relabelling for
  a permutation among global qubits), then read shard by shard in chunks.
"""
from __future__ import annotations

import numpy as np

from .circuit import Circuit, GateKind, GateOp, as_precision
from .sharded import LocalStep, SwapStep, _schedule_once, block_peer, localize, own_block, schedule

class ShardedDeviceState:
    """A 2^n state sharded over the devices of this process (see module doc)."""

    def __init__(self, engine, num_qubits: int, precision, shards: list, layout: list):
        self.num_qubits = num_qubits
        self.precision = precision
        self.shards = shards          # DeviceStateVector per rank, rank r = global bits r
        self.layout = list(layout)    # phys_of[logical qubit]
        self._engine = engine
        self._host = None
        self._host_version = -1
        self._version = 0

    @property
    def world(self) -> int:
        return len(self.shards)

    @property
    def g(self) -> int:
        return self.world.bit_length() - 1

    @property
    def n_local(self) -> int:
        return self.num_qubits - self.g

    def touch(self) -> None:
        self._version += 1
        for s in self.shards:
            s.touch()

    def synchronize(self) -> None:
        for s in self.shards:
            s._engine.synchronize()

    @property
    def amplitudes(self) -> np.ndarray:
        """Logical little-endian amplitudes on the host (identity layout restored
        on the device first; each shard copied in pinned, chunked pieces)."""
        from .b200 import d2h_chunked
        if self._host is None or self._host_version != self._version:
            canonicalize(self)
            self.synchronize()
            self._host = None
            L = 1 << self.n_local
            out = np.empty(L * self.world, dtype=as_precision(self.precision).dtype)
            for r, sh in enumerate(self.shards):
                d2h_chunked(sh.tensor, out[r * L:(r + 1) * L])
            self._host = out
            self._host_version = self._version
        return self._host

    def norm_squared(self) -> float:
        return float(sum(s._engine.norm_squared(s) for s in self.shards))

    def probabilities(self) -> np.ndarray:
        canonicalize(self)
        return np.concatenate([s._engine.probabilities(s) for s in self.shards])


# ------------------------------------------------------------------ execution

def _shard_engines(engine, devices):
    return [engine.device_engine(d) for d in devices]


def init_sharded(engine, num_qubits: int, precision, devices) -> ShardedDeviceState:
    """|0...0> over len(devices) shards (rank 0 holds amplitude 0)."""
    import ctypes as C

    from . import _native
    from .b200 import prec_code
    world = len(devices)
    g = world.bit_length() - 1
    if 1 << g != world:
        raise ValueError("the shard count must be a power of two")
    nl = num_qubits - g
    if nl < 1:
        raise ValueError("too many shards for the qubit count")
    shards = []
    for r, eng in enumerate(_shard_engines(engine, devices)):
        st = eng.init_state(nl, precision)
        if r:
            _native.check(_native.lib().svb_fill_basis(C.c_void_p(st.tensor.data_ptr()), nl,
                                                       prec_code(precision), -1, C.c_void_p(eng.stream())))
        shards.append(st)
    return ShardedDeviceState(engine, num_qubits, precision, shards, list(range(num_qubits)))


def _run_local(state: ShardedDeviceState, gates) -> None:
    if not gates:
        return
    nl = state.n_local
    for r, sh in enumerate(state.shards):
        eng = sh._engine
        mine = localize(gates, nl, r)
        eng.execute(sh, eng.plan(Circuit(nl, mine), state.precision))


def exchange(state: ShardedDeviceState, step: SwapStep) -> None:
    """Swap the step's global qubits with the top m local qubits: shard r's
    block own(p) <-> shard p's block own(r) for every partner p (the same
    pairing as the torchrun path, sharded.ShardedEngine.exchange).

    Each pair of blocks is swapped IN PLACE by the swap kernel
    (svb_swap_blocks): shard r's device swaps the first half of the pair and
    shard p's device the second half, concurrently, each reading and writing
    the other GPU's half through peer access (NVLink) -- no staging buffer,
    no extra device copy, both link directions busy."""
    import torch

    from . import _native
    state.synchronize()
    nl = step.n_local
    blk = 1 << (nl - step.m)
    esz = state.shards[0].tensor.element_size()
    done = set()
    used = set()
    for r in range(state.world):
        for w in range(1 << step.m):
            if w == own_block(r, step):
                continue
            p = block_peer(r, step, w)
            if (min(r, p), max(r, p)) in done:
                continue
            done.add((min(r, p), max(r, p)))
            ta, tb = state.shards[r].tensor, state.shards[p].tensor
            wa, wb = own_block(p, step), own_block(r, step)
            a0 = ta.data_ptr() + wa * blk * esz
            b0 = tb.data_ptr() + wb * blk * esz
            total = blk * esz
            if total % 16:  # a single c64 amplitude per block (tiny states)
                sa, sb = ta[wa * blk:(wa + 1) * blk], tb[wb * blk:(wb + 1) * blk]
                tmp = sa.clone()
                sa.copy_(sb.to(sa.device))
                sb.copy_(tmp.to(sb.device))
                used.update((ta.device, tb.device))
                continue
            half = (total // 2) // 16 * 16
            for dev, lo, hi in ((ta.device, 0, half), (tb.device, half, total)):
                if hi <= lo:
                    continue
                if ta.device != tb.device:
                    other = tb.device if dev == ta.device else ta.device
                    _native.enable_peer_access(dev.index, other.index)
                with torch.cuda.device(dev):
                    _native.swap_blocks(a0 + lo, b0 + lo, hi - lo, torch.cuda.current_stream(dev).cuda_stream)
                used.add(dev)
    for dev in used:
        torch.cuda.synchronize(dev)
    for s in state.shards:
        s.touch()


def run_schedule(state: ShardedDeviceState, sched) -> ShardedDeviceState:
    for st in sched.steps:
        if isinstance(st, LocalStep):
            _run_local(state, st.gates)
        else:
            exchange(state, st)
    state.layout = list(sched.final_layout)
    state.touch()
    return state


def run_circuit_sharded(engine, circuit, precision, devices) -> ShardedDeviceState:
    """Fresh |0...0> over the devices, then the whole circuit: the initial
    layout may be any relabelling (|0...0> is invariant), chosen so the first
    swap needs no SWAP gates (sharded.schedule)."""
    sched = schedule(circuit, len(devices))
    state = init_sharded(engine, circuit.num_qubits, precision, devices)
    state.layout = list(sched.initial_layout)
    return run_schedule(state, sched)


def apply_sharded(state: ShardedDeviceState, gates) -> ShardedDeviceState:
    """Gates on the state's current layout (the per-gate / checkpoint path)."""
    sched, _ = _schedule_once(list(gates), state.num_qubits, state.g, state.layout)
    return run_schedule(state, sched)


def canonicalize(state: ShardedDeviceState) -> None:
    """Move data so that logical qubit q is physical qubit q (identity layout)."""
    n, nl = state.num_qubits, state.n_local
    phys = list(state.layout)
    if phys == list(range(n)):
        return
    log_at = [0] * n
    for q, p in enumerate(phys):
        log_at[p] = q

    def local_swap(a: int, b: int, batch: list):
        batch.append(GateOp(GateKind.SWAP, (min(a, b), max(a, b))))
        qa, qb = log_at[a], log_at[b]
        phys[qa], phys[qb] = b, a
        log_at[a], log_at[b] = qb, qa

    # A: every logical qubit >= nl onto a global position
    for gp in range(nl, n):
        if log_at[gp] >= nl:
            continue
        q = next(q for q in range(nl, n) if phys[q] < nl)
        batch: list = []
        if phys[q] != nl - 1:
            local_swap(phys[q], nl - 1, batch)
        _run_local(state, batch)
        exchange(state, SwapStep([gp], nl))
        qa, qb = log_at[nl - 1], log_at[gp]
        phys[qa], phys[qb] = gp, nl - 1
        log_at[nl - 1], log_at[gp] = qb, qa
    # B: a permutation among the global qubits relabels the shards
    if any(phys[q] != q for q in range(nl, n)):
        new = [None] * state.world
        for r in range(state.world):
            # shard r holds global physical bits r; logical bit (q - nl) of its
            # new rank is the physical bit phys[q] - nl of r
            r2 = 0
            for q in range(nl, n):
                r2 |= ((r >> (phys[q] - nl)) & 1) << (q - nl)
            new[r2] = state.shards[r]
        state.shards = new
        for q in range(nl, n):
            log_at[q] = q
            phys[q] = q
    # C: local permutation as physical SWAP gates in one plan per shard
    batch = []
    for p in range(nl):
        if log_at[p] != p:
            local_swap(phys[p], p, batch)
    _run_local(state, batch)
    state.layout = list(range(n))
    state.touch()


def plan_shards(engine, num_qubits: int, precision, devices) -> int:
    """Shards needed: 1 when the state fits the first device, else the
    smallest power of two whose shards fit every device used (-1: none)."""
    import torch
    need = (1 << num_qubits) * as_precision(precision).amplitude_bytes
    world = 1
    while world <= len(devices):
        per = need // world
        ok = True
        for d in devices[:world]:
            free, _ = torch.cuda.mem_get_info(d)
            # a shard of the same device may already hold memory: count it once
            ok = ok and per + (256 << 20) <= free / max(1, devices[:world].count(d))
        if ok and (num_qubits - (world.bit_length() - 1)) >= 1:
            return world
        world *= 2
    return -1
