"""State-vector sharding over P = 2^g GPUs with global-qubit swaps.

The reference runs one process on one device and, when a state does not fit,
falls back to the CPU (ref ``pkg/src/aqsim/memory.py:290-340``).  Here the
state is partitioned instead: rank r holds the 2^(n-g) amplitudes whose top g
*physical* index bits equal r, so physical qubits n-g..n-1 are "global".

The scheduler keeps a logical<->physical qubit permutation (allowed by the
reference contract that engines may swap buffers between gates,
ref ``circuit.py:189-194``):

* a *local segment* is every pending gate whose qubits are all local and that
  no deferred gate must precede (same dependency rule as the planner); it runs
  as one planned sequence of tile passes on each shard.  Diagonal gates join
  a segment even when they touch global qubits: a global bit is constant on a
  rank, so each rank applies the diagonal restricted to its own global bits
  (``localize``) -- diagonal gates never cause an exchange;
* a *swap* brings the global qubits the next deferred gates need into the top
  m local positions: each rank splits its shard into 2^m contiguous blocks by
  those m bits and exchanges block w with the rank whose global bits equal w
  (an all-to-all inside groups of 2^m ranks; the rank's own block stays);
* victims (local qubits sent out) are the ones used furthest in the future;
  they are moved to the top local positions by physical SWAP gates folded into
  the preceding segment, and the *initial* layout is chosen so that the first
  swap needs none (|0...0> is invariant under qubit relabelling).

Transport on the GPU box (``p2p``, the default for CUDA shards): every rank
maps its peers' shards into its address space once (CUDA IPC handles
exchanged over ``torch.distributed``) and a swap is ONE kernel per rank
(``svb_swap_blocks``): for each block pair the lower rank swaps the first
half and the higher rank the second half, loading and storing the peer's
memory over NVLink -- in place, no staging buffer, no copy-back.  The
fallback (``p2p=False``, and the CPU tests) is ``torch.distributed``
point-to-point chunked through a double-buffered staging area so that the
copy-back of chunk c overlaps the transfer of chunk c+1.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .circuit import GateKind, GateOp, Precision, as_precision, effective_unitary


# --------------------------------------------------------------- scheduling

@dataclass
class LocalStep:
    gates: list                      # GateOps with PHYSICAL local targets


@dataclass
class SwapStep:
    global_pos: list                 # physical global positions (ascending), each >= n_local
    n_local: int

    @property
    def m(self) -> int:
        return len(self.global_pos)

    @property
    def local_pos(self) -> list:
        return [self.n_local - self.m + i for i in range(self.m)]


@dataclass
class Schedule:
    n: int
    g: int
    initial_layout: list             # phys_of[logical]
    final_layout: list
    steps: list = field(default_factory=list)

    @property
    def n_local(self) -> int:
        return self.n - self.g

    def num_swaps(self) -> int:
        return sum(isinstance(s, SwapStep) for s in self.steps)


def _physical_op(op, phys_of) -> GateOp:
    return GateOp(GateKind.CUSTOM, tuple(phys_of[t] for t in op.targets), (), effective_unitary(op))


def _is_diagonal(op) -> bool:
    u = effective_unitary(op)
    return not np.any(u - np.diag(np.diag(u)))


def localize(gates, n_local: int, rank: int) -> list:
    """Specialise a local segment to one rank: a diagonal gate on physical
    qubits >= n_local (global) keeps only its local qubits, its entries taken
    at this rank's global bits; a diagonal on global qubits only becomes a
    constant phase of the shard (a 1-qubit diagonal on qubit 0)."""
    out = []
    for op in gates:
        tg = tuple(op.targets)
        if all(t < n_local for t in tg):
            out.append(op)
            continue
        d = np.diag(effective_unitary(op))
        loc = [j for j, t in enumerate(tg) if t < n_local]
        fixed = sum(((rank >> (t - n_local)) & 1) << j for j, t in enumerate(tg) if t >= n_local)
        sub = np.empty(1 << len(loc), dtype=np.complex128)
        for x in range(sub.size):
            sub[x] = d[fixed | sum(((x >> k) & 1) << j for k, j in enumerate(loc))]
        if loc:
            out.append(GateOp(GateKind.CUSTOM, tuple(tg[j] for j in loc), (), np.diag(sub)))
        else:
            out.append(GateOp(GateKind.CUSTOM, (0,), (), np.diag([sub[0], sub[0]])))
    return out


def _schedule_once(gates, n: int, g: int, layout: list) -> tuple[Schedule, list]:
    nl = n - g
    phys_of = list(layout)
    log_at = [0] * n
    for q, p in enumerate(phys_of):
        log_at[p] = q
    sched = Schedule(n, g, list(layout), [])
    pending = list(range(len(gates)))
    first_victims: list = []
    diag = [_is_diagonal(op) for op in gates]
    while pending:
        blocked: set = set()
        seg, deferred = [], []
        for i in pending:
            tg = gates[i].targets
            if any(t in blocked for t in tg) or (not diag[i] and any(phys_of[t] >= nl for t in tg)):
                deferred.append(i)
                blocked.update(tg)
            else:
                seg.append(_physical_op(gates[i], phys_of))
        if seg:
            sched.steps.append(LocalStep(seg))
        if not deferred:
            break
        # global logical qubits the deferred gates need, in first-use order
        need: list = []
        for i in deferred:
            for t in gates[i].targets:
                if phys_of[t] >= nl and t not in need:
                    need.append(t)
        m = min(len(need), g)
        need = need[:m]
        first_tg = set(gates[deferred[0]].targets)
        if not set(t for t in first_tg if phys_of[t] >= nl) <= set(need):
            raise RuntimeError("scheduler: first deferred gate needs more global qubits than exist")
        # victims: local logical qubits not needed by the first deferred gate,
        # with the furthest next use
        next_use = {}
        for pos, i in enumerate(deferred):
            for t in gates[i].targets:
                next_use.setdefault(t, pos)
        cands = [log_at[p] for p in range(nl) if log_at[p] not in first_tg]
        if len(cands) < m:
            raise ValueError("not enough local qubits for a global swap (n_local too small)")
        cands.sort(key=lambda q: (-next_use.get(q, len(deferred) + 1), -phys_of[q]))
        victims = cands[:m]
        if not first_victims:
            first_victims = list(victims)
        top = [nl - m + i for i in range(m)]
        # move victims onto the top local positions with physical SWAPs
        fix = []
        placed = [v for v in victims if phys_of[v] in top]
        free_top = [p for p in top if log_at[p] not in placed]
        for v in victims:
            if v in placed:
                continue
            p_dst = free_top.pop(0)
            a, b = phys_of[v], p_dst
            fix.append(GateOp(GateKind.SWAP, (min(a, b), max(a, b))))
            qa, qb = log_at[a], log_at[b]
            phys_of[qa], phys_of[qb] = b, a
            log_at[a], log_at[b] = qb, qa
        if fix:
            if sched.steps and isinstance(sched.steps[-1], LocalStep):
                sched.steps[-1].gates.extend(fix)
            else:
                sched.steps.append(LocalStep(fix))
        # pair victim at top position i with the i-th ascending global position
        gpos = sorted(phys_of[q] for q in need)
        sched.steps.append(SwapStep(gpos, nl))
        for i, gp in enumerate(gpos):
            lp = nl - m + i
            qa, qb = log_at[lp], log_at[gp]
            phys_of[qa], phys_of[qb] = gp, lp
            log_at[lp], log_at[gp] = qb, qa
        pending = deferred
    sched.final_layout = list(phys_of)
    return sched, first_victims


def schedule(circuit, world_size: int, optimise_layout: bool = True) -> Schedule:
    """Lower a (fused) circuit into local segments and global swaps."""
    n = circuit.num_qubits
    g = int(round(math.log2(world_size)))
    if 1 << g != world_size:
        raise ValueError("world size must be a power of two")
    if g > n - 1:
        raise ValueError("too many ranks for the qubit count")
    gates = list(circuit.gates)
    ident = list(range(n))
    sched, victims = _schedule_once(gates, n, g, ident)
    if g == 0 or not optimise_layout or not victims:
        return sched
    # initial layout: first-swap victims start on the top local positions
    layout = list(ident)
    log_at = list(range(n))
    nl = n - g
    top = [nl - len(victims) + i for i in range(len(victims))]
    for v, p_dst in zip(victims, top):
        a = layout[v]
        if a == p_dst:
            continue
        qb = log_at[p_dst]
        layout[v], layout[qb] = p_dst, a
        log_at[a], log_at[p_dst] = qb, v
    better, _ = _schedule_once(gates, n, g, layout)
    swaps_a = sum(len(s.gates) for s in sched.steps if isinstance(s, LocalStep))
    swaps_b = sum(len(s.gates) for s in better.steps if isinstance(s, LocalStep))
    if (better.num_swaps(), swaps_b) <= (sched.num_swaps(), swaps_a):
        return better
    return sched


def block_peer(rank: int, step: SwapStep, w: int) -> int:
    """Rank that exchanges block w with `rank` in a swap."""
    r = rank
    for i, gp in enumerate(step.global_pos):
        j = gp - step.n_local
        r = (r & ~(1 << j)) | (((w >> i) & 1) << j)
    return r


def own_block(rank: int, step: SwapStep) -> int:
    return sum(((rank >> (gp - step.n_local)) & 1) << i for i, gp in enumerate(step.global_pos))


def unpermute(full_physical: np.ndarray, n: int, phys_of: list) -> np.ndarray:
    """Physical-order amplitudes -> logical little-endian order."""
    t = full_physical.reshape((2,) * n)          # axis a <-> physical bit n-1-a
    # logical axis order (big-endian): logical bit n-1-a' at axis a'
    axes = [n - 1 - phys_of[n - 1 - a] for a in range(n)]
    return np.ascontiguousarray(t.transpose(axes)).reshape(-1)


# ----------------------------------------------------------------- execution

class CudaShardBackend:
    """Local work on a shard through libsvb200 (the product path)."""

    def __init__(self, device, options=None):
        import torch
        from .b200 import B200Engine
        self.torch = torch
        self.engine = B200Engine("b200-shard", device=device, options=options)
        self.device = self.engine.device

    def alloc(self, n_local: int, precision):
        state = self.engine.init_state(n_local, precision)
        return state

    def fill(self, state, index_of_one: int):
        import ctypes as C
        from . import _native
        from .b200 import prec_code
        _native.check(_native.lib().svb_fill_basis(
            C.c_void_p(state.tensor.data_ptr()), state.num_qubits, prec_code(state.precision),
            index_of_one, C.c_void_p(self.engine.stream())))
        state.touch()

    def plan(self, n_local: int, precision, gates):
        from .b200 import CircuitPlan
        return CircuitPlan(n_local, precision, gates, self.engine.options)

    def run(self, state, plan):
        self.engine.execute(state, plan)

    def tensor(self, state):
        return state.tensor

    def norm2(self, state) -> float:
        return self.engine.norm_squared(state)

    def synchronize(self):
        self.engine.synchronize()


class ShardedEngine:
    """Runs circuits on a state sharded over the torch.distributed world."""

    def __init__(self, backend, group=None, chunk_elems: int = 1 << 24, p2p: bool | None = None):
        import torch.distributed as dist
        self.dist = dist
        self.backend = backend
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.chunk_elems = chunk_elems
        self._staging = None
        # None: peer-mapped swap kernel when the shards are CUDA tensors under
        # NCCL (one node); True forces it (e.g. gloo ranks sharing one GPU)
        self.p2p = p2p
        self._peers = {}   # peer allocation's IPC handle -> mapped base
        self._bases = []   # IPC mappings to close

    def close(self) -> None:
        from . import _native
        for b in self._bases:
            try:
                _native.ipc_close(b)
            except Exception:  # pragma: no cover - teardown
                pass
        self._bases = []
        self._peers = {}

    def _use_p2p(self, t) -> bool:
        if not t.is_cuda:
            return False
        if self.p2p is not None:
            return bool(self.p2p)
        return self.dist.get_backend(self.group) == "nccl"

    def _peer_ptrs(self, t) -> dict:
        """Every rank's shard mapped into this process (CUDA IPC).  Handles
        are gathered at every exchange (a re-allocated shard gets a new
        handle even at a recycled address); mappings are cached per handle."""
        import torch

        from . import _native
        try:
            mine = _native.ipc_export(t.data_ptr())
        except Exception:  # e.g. a driver without IPC: every rank falls back together
            mine = None
        allh = [None] * self.world
        self.dist.all_gather_object(allh, mine, group=self.group)
        ptrs, ok = {}, all(x is not None for x in allh)
        for r, hx in enumerate(allh if ok else []):
            h, off = hx
            if r == self.rank:
                ptrs[r] = t.data_ptr()
                continue
            try:
                if h not in self._peers:
                    _ptr, base = _native.ipc_import(h, 0)
                    self._peers[h] = base
                    self._bases.append(base)
                ptrs[r] = self._peers[h] + off
            except Exception:
                ok = False
                break
        # every rank must agree (a one-sided fallback would deadlock the swap)
        dev = t.device if self.dist.get_backend(self.group) == "nccl" else torch.device("cpu")
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        self.dist.all_reduce(flag, op=self.dist.ReduceOp.MIN, group=self.group)
        return ptrs if int(flag.item()) == 1 else None

    def _exchange_p2p_step(self, t, step, blk: int, peers) -> bool:
        """Block swaps as one kernel per rank over peer-mapped memory: the pair
        (our block w, peer's block own(rank)) is split in halves, the lower
        rank swaps the first, the higher the second, both at once.  False when
        some rank cannot map its peers (the caller falls back to NCCL)."""
        import torch

        from . import _native
        ptrs = self._peer_ptrs(t)
        if ptrs is None:
            return False
        esz = t.element_size()
        total = blk * esz
        half = (total // 2) // 16 * 16
        stream = torch.cuda.current_stream(t.device).cuda_stream
        torch.cuda.synchronize(t.device)    # this shard's earlier passes are done ...
        self.dist.barrier(group=self.group)  # ... and every peer's
        mine = own_block(self.rank, step)   # where our block w lands on the peer
        for w, peer in peers:
            a0 = t.data_ptr() + w * total
            b0 = ptrs[peer] + mine * total
            lo, hi = (0, half) if self.rank < peer else (half, total)
            if hi > lo:
                _native.swap_blocks(a0 + lo, b0 + lo, hi - lo, stream)
        torch.cuda.synchronize(t.device)    # our half of every pair is swapped ...
        self.dist.barrier(group=self.group)  # ... and the peers' halves
        return True

    # -------------------------------------------------------------- program
    def compile(self, circuit, precision=Precision.DOUBLE):
        precision = as_precision(precision)
        sched = schedule(circuit, self.world)
        progs = []
        for st in sched.steps:
            if isinstance(st, LocalStep):
                gates = localize(st.gates, sched.n_local, self.rank)
                progs.append(("local", self.backend.plan(sched.n_local, precision, gates)))
            else:
                progs.append(("swap", st))
        return sched, progs

    def init_state(self, n_local: int, precision):
        state = self.backend.alloc(n_local, precision)
        self.backend.fill(state, 0 if self.rank == 0 else -1)
        return state

    def run_program(self, state, progs):
        for kind, obj in progs:
            if kind == "local":
                self.backend.run(state, obj)
            else:
                self.exchange(state, obj)
        return state

    def run_circuit(self, circuit, precision=Precision.DOUBLE):
        sched, progs = self.compile(circuit, precision)
        state = self.init_state(sched.n_local, precision)
        self.run_program(state, progs)
        self.backend.synchronize()
        return ShardedState(self, state, sched)

    # ------------------------------------------------------------- exchange
    def _staging_for(self, t, elems: int):
        if self._staging is None or self._staging.numel() < elems or self._staging.dtype != t.dtype \
                or self._staging.device != t.device:
            self._staging = t.new_empty(elems)
        return self._staging[:elems]

    def exchange(self, state, step: SwapStep):
        """Swap the step's global qubits with the top m local qubits (in place)."""
        dist = self.dist
        t = self.backend.tensor(state)
        nl = step.n_local
        m = step.m
        blk = 1 << (nl - m)
        chunk = min(blk, self.chunk_elems)
        n_chunks = blk // chunk
        mine = own_block(self.rank, step)
        peers = [(w, block_peer(self.rank, step, w)) for w in range(1 << m) if w != mine]
        if not peers:
            return
        npeer = len(peers)
        if self._use_p2p(t) and (blk * t.element_size()) % 16 == 0:
            if self._exchange_p2p_step(t, step, blk, peers):
                if hasattr(state, "touch"):
                    state.touch()
                return
            self.p2p = False  # IPC unavailable on some rank: NCCL point-to-point from now on
        if t.is_cuda and dist.get_backend(self.group) == "gloo":
            # gloo moves host tensors only (used by the single-GPU multi-process
            # tests): stage each block through host memory
            self._exchange_via_host(t, blk, mine, peers)
            if hasattr(state, "touch"):
                state.touch()
            return
        stage = self._staging_for(t, 2 * npeer * chunk).view(2, npeer, chunk)

        def issue(c):
            ops = []
            for k, (w, peer) in enumerate(peers):
                src = t[w * blk + c * chunk: w * blk + (c + 1) * chunk]
                ops.append(dist.P2POp(dist.isend, src, peer, self.group))
                ops.append(dist.P2POp(dist.irecv, stage[c % 2, k], peer, self.group))
            return dist.batch_isend_irecv(ops)

        inflight = issue(0)
        for c in range(n_chunks):
            nxt = issue(c + 1) if c + 1 < n_chunks else None
            for r in inflight:
                r.wait()
            for k, (w, _peer) in enumerate(peers):
                t[w * blk + c * chunk: w * blk + (c + 1) * chunk].copy_(stage[c % 2, k])
            inflight = nxt
        if hasattr(state, "touch"):
            state.touch()


    def _exchange_via_host(self, t, blk: int, mine: int, peers):
        dist = self.dist
        ops, recv = [], []
        for w, peer in peers:
            src = t[w * blk:(w + 1) * blk].cpu()
            buf = torch_empty_like_host(src)
            ops.append(dist.P2POp(dist.isend, src, peer, self.group))
            ops.append(dist.P2POp(dist.irecv, buf, peer, self.group))
            recv.append((w, buf))
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        for w, buf in recv:
            t[w * blk:(w + 1) * blk].copy_(buf)


def torch_empty_like_host(x):
    import torch
    return torch.empty_like(x, device="cpu")


class ShardedState:
    """Handle on a sharded result: device reductions and (small n) gathering."""

    def __init__(self, engine: ShardedEngine, state, sched: Schedule):
        self.engine = engine
        self.state = state
        self.schedule = sched
        self.num_qubits = sched.n

    def _reduce_device(self):
        """Device of the reduction tensors: the shard's own GPU under NCCL (an
        NCCL-only group has no CPU backend), host memory otherwise."""
        import torch
        if self.engine.dist.get_backend(self.engine.group) == "nccl":
            return self.engine.backend.tensor(self.state).device
        return torch.device("cpu")

    def norm_squared(self) -> float:
        import torch
        v = torch.tensor([self.engine.backend.norm2(self.state)], dtype=torch.float64,
                         device=self._reduce_device())
        self.engine.dist.all_reduce(v, group=self.engine.group)
        return float(v.item())

    def gather(self) -> np.ndarray | None:
        """Full logical-order state on rank 0 (None elsewhere); for modest n."""
        import torch
        dist = self.engine.dist
        t = self.engine.backend.tensor(self.state).detach()
        host = t.cpu() if t.device.type != "cpu" else t
        if dist.get_backend(self.engine.group) == "nccl":
            parts = [torch.empty_like(t) for _ in range(self.engine.world)]
            dist.all_gather(parts, t, group=self.engine.group)
            parts = [p.cpu() for p in parts]
        else:
            parts = [torch.empty_like(host) for _ in range(self.engine.world)]
            dist.all_gather(parts, host.contiguous(), group=self.engine.group)
        if self.engine.rank != 0:
            return None
        full = torch.cat(parts).numpy()
        return unpermute(full, self.schedule.n, self.schedule.final_layout)
