"""CPU checks of the native planner (libsvb200.so, host-only entry points).

1. Legality: executing the input gates in the order the plan applies them
   (pass by pass) gives the oracle's program-order state.
2. Lowering: a numpy emulation of what k_tile_pass does with each pass
   (tile gather by L/high bits, kernel ops on tile-local bits with the
   planner's merged coefficients, scatter) reproduces the oracle state.
3. Error behaviour mirrors the reference (ValueError on bad targets).
"""
from __future__ import annotations

import numpy as np
import pytest

from golden_io import decode
from oracle import sv_oracle as orc
from paper_2604_03816_b200 import generators as gen
from paper_2604_03816_b200.b200 import CircuitPlan, plan_options
from paper_2604_03816_b200.circuit import Circuit, GateKind, GateOp, Precision
from paper_2604_03816_b200.fusion import fuse


def tile_indices(n: int, info: dict, tile: int) -> np.ndarray:
    """Global amplitude index of every tile-local index (the kernel's addressing)."""
    L, high, T = info["low_bits"], info["high"], info["tile_bits"]
    g = tile << L
    for p in sorted(high):
        g = ((g >> p) << (p + 1)) | (g & ((1 << p) - 1))
    local = np.arange(1 << T)
    idx = np.full(1 << T, g, dtype=np.int64) + (local & ((1 << L) - 1))
    for b, p in enumerate(high):
        idx += ((local >> (L + b)) & 1) << p
    return idx


def emulate(plan: CircuitPlan, n: int, precision: str) -> np.ndarray:
    amps = orc.init_state(n, precision)
    nat = plan.native
    for p in range(nat.num_passes()):
        emulate_tile_pass(amps, nat, p, n)
    return amps


def emulate_tile_pass(amps: np.ndarray, nat, p: int, n: int) -> None:
    """One pass as k_tile_pass runs it (tile gather, ops on tile bits, scatter)."""
    if True:
        info = nat.pass_info(p)
        T = info["tile_bits"]
        ops = [nat.kernel_op(p, i) for i in range(info["num_kernel_ops"])]
        for tile in range(1 << (n - T)):
            idx = tile_indices(n, info, tile)
            buf = amps[idx].copy()
            for op in ops:
                if op["kind"] == "dense":
                    u = op["coeffs"].reshape(1 << op["k"], 1 << op["k"])
                    orc.apply_matrix(buf, T, op["targets"], u)
                elif op["kind"] == "ctrl":  # U0 / U1 on a tile bit, control = shard qubit outside the tile
                    sel = int(idx[0] >> op["ctrl_qubit"]) & 1
                    u = op["coeffs"].reshape(2, 2, 2)[sel]
                    orc.apply_matrix(buf, T, op["targets"], u)
                elif op["kind"] == "perm":  # CNOT(control, target) on tile bits
                    c_, t_ = op["targets"]
                    e = np.arange(1 << T)
                    sel = ((e >> c_) & 1).astype(bool) & ~((e >> t_) & 1).astype(bool)
                    a_, b_ = e[sel], e[sel] | (1 << t_)
                    buf[a_], buf[b_] = buf[b_].copy(), buf[a_].copy()
                else:
                    d = np.zeros(1 << T, dtype=np.int64)
                    e = np.arange(1 << T)
                    for b, t in enumerate(op["targets"]):
                        # t >= T: shard qubit t - T outside the tile (per-tile constant)
                        d |= (((e >> t) if t < T else (idx >> (t - T))) & 1) << b
                    buf *= op["coeffs"].astype(buf.dtype)[d]
            amps[idx] = buf


def plan_order_state(plan: CircuitPlan, circuit, precision: str) -> np.ndarray:
    amps = orc.init_state(circuit.num_qubits, precision)
    seen = []
    for p in range(plan.native.num_passes()):
        for gi in plan.native.pass_gates(p):
            orc.apply_gate(amps, circuit.num_qubits, circuit.gates[gi])
            seen.append(gi)
    assert sorted(seen) == list(range(len(circuit.gates)))
    return amps


CASES = [
    ("layered8", lambda: fuse(gen.layered_circuit(8, layers=6), 2)[0]),
    ("layered9_w3", lambda: fuse(gen.layered_circuit(9, layers=5, seed=2), 3)[0]),
    ("qft9", lambda: fuse(gen.qft_circuit(9), 2)[0]),
    ("qft8_raw", lambda: gen.qft_circuit(8)),
    ("su2", lambda: gen.random_su2_circuit(7, 60, seed=4)),
]
OPTIONS = [
    {},
    {"tile_bits": 5, "min_low_bits": 2},
    {"tile_bits": 4, "min_low_bits": 1, "cost_budget": -1.0},
    {"tile_bits": 6, "min_low_bits": 3, "no_diag_merge": 1},
    {"tile_bits": 5, "min_low_bits": 1, "max_ops_per_pass": 2},
]


@pytest.mark.parametrize("name,make", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("opts", OPTIONS, ids=[str(o) for o in OPTIONS])
def test_plan_legal_and_lowering(name, make, opts):
    c = make()
    want = orc.run_circuit(c, "double")
    plan = CircuitPlan(c.num_qubits, Precision.DOUBLE, c.gates, plan_options(**opts) if opts else None)
    assert np.abs(plan_order_state(plan, c, "double") - want).max() <= 1e-12
    assert np.abs(emulate(plan, c.num_qubits, "double") - want).max() <= 1e-12
    # single precision plans round coefficients like ref engines.py:157
    plan1 = CircuitPlan(c.num_qubits, Precision.SINGLE, c.gates, plan_options(**opts) if opts else None)
    got = emulate(plan1, c.num_qubits, "single")
    assert np.abs(got - want).max() <= 1e-5


def test_plan_golden_random_circuits(golden_random):
    for i in range(int(golden_random["count"])):
        c = decode(f"c{i}_", golden_random)
        plan = CircuitPlan(c.num_qubits, Precision.DOUBLE, c.gates,
                           plan_options(tile_bits=min(4, c.num_qubits), min_low_bits=1))
        got = emulate(plan, c.num_qubits, "double")
        assert np.abs(got - golden_random[f"c{i}_c128"]).max() <= 1e-12, i


def test_plan_structure_layered28():
    f, _ = fuse(gen.layered_circuit(28), 2)
    for prec in (Precision.SINGLE, Precision.DOUBLE):
        plan = CircuitPlan(28, prec, f.gates)
        passes = plan.passes()
        assert sum(p["num_gates"] for p in passes) == len(f.gates) == 189
        assert len(passes) < len(f.gates) / 2
        for p in passes:
            assert p["low_bits"] + len(p["high"]) == p["tile_bits"]
            assert p["low_bits"] >= (4 if prec is Precision.SINGLE else 3)
            assert p["reg_bits"] == (5 if prec is Precision.SINGLE else 4)
            assert p["tile_bits"] == 12 if prec is Precision.SINGLE else 11


def test_diagonal_runs_are_merged_qft():
    f, _ = fuse(gen.qft_circuit(20), 2)
    plan = CircuitPlan(20, Precision.DOUBLE, f.gates)
    n_ops = sum(p["num_kernel_ops"] for p in plan.passes())
    assert n_ops < len(f.gates) / 2


def test_planner_errors():
    with pytest.raises(ValueError):
        CircuitPlan(3, Precision.DOUBLE, [GateOp(GateKind.X, (3,))])
    with pytest.raises(ValueError):
        CircuitPlan(0, Precision.DOUBLE, [])
    wide = GateOp(GateKind.CUSTOM, tuple(range(7)), (), np.eye(128))
    with pytest.raises(ValueError):
        CircuitPlan(8, Precision.DOUBLE, [wide])


def test_empty_and_single_qubit_states():
    plan = CircuitPlan(1, Precision.SINGLE, [GateOp(GateKind.H, (0,))])
    assert plan.num_passes == 1
    got = emulate(plan, 1, "single")
    assert np.allclose(got, [2 ** -0.5, 2 ** -0.5], atol=1e-7)
    assert CircuitPlan(3, Precision.DOUBLE, []).num_passes == 0


# ---------------------------------------------------------------------------
# register-phase encoding (k_reg_pass semantics, swizzle omitted: it is a
# bijection applied identically on both sides of every transpose)

def _deposit(x: int, mask: int, rb: int) -> int:
    r, b = 0, 0
    for i in range(rb):
        if (mask >> i) & 1:
            if (x >> b) & 1:
                r |= 1 << i
            b += 1
    return r


def emulate_reg(plan: CircuitPlan, n: int, precision: str) -> np.ndarray:
    amps = orc.init_state(n, precision)
    nat = plan.native
    for p in range(nat.num_passes()):
        info = nat.pass_info(p)
        T, rb = info["tile_bits"], info["reg_bits"]
        if rb == 0 and info["kernel"] == "tile":  # a shared-memory pass inside a register plan
            emulate_tile_pass(amps, nat, p, n)
            continue
        assert rb > 0 and T - rb in (7, 8)
        nr = 1 << rb
        nthreads = 1 << (T - rb)
        phases = [nat.phase(p, f) for f in range(info["num_phases"])]
        ops = [nat.phase_op(p, i) for i in range(info["num_kernel_ops"])]
        tid = np.arange(nthreads)
        for tile in range(1 << (n - T)):
            idx = tile_indices(n, info, tile)
            buf = amps[idx].copy()
            for ph in phases:
                R = ph["R"][:rb]
                mp = ph["map"]
                if info["kernel"] == "gemm":
                    # k_gemm_pass: the GEMM acts on the column qubits R (matrix
                    # order), then the diagonal ops in the read-out layout `map`
                    if ph["tc"] >= 0:
                        gm = list(R) + [q for q in range(T) if q not in R]
                        base = np.zeros(nthreads, dtype=np.int64)
                        for k in range(T - rb):
                            base |= ((tid >> k) & 1) << gm[rb + k]
                        cl = np.stack([base + sum(1 << gm[i] for i in range(rb) if (rho >> i) & 1)
                                       for rho in range(nr)], axis=1)
                        U = nat.tc_matrix(p, ph["tc"]).astype(buf.dtype)
                        buf[cl] = buf[cl] @ U.T
                    ph = dict(ph, tc=-1, op_mid=ph["op_begin"])
                assert sorted(mp[:T]) == list(range(T)), mp  # the layout is a bit permutation
                if ph["mma"] and T - rb == 8:
                    # fragment layout (svb_regpass.cuh mma_phase): K bits R[2..4] in
                    # registers 0..2, R[0..1] in lanes 0..1; the GEMM acts on R
                    assert mp[0:3] == R[2:5] and mp[5:7] == R[0:2], (mp, R)
                    assert ph["op_begin"] == ph["op_end"]
                    mp = list(R) + [q for q in range(T) if q not in R]
                elif ph["mma"]:
                    # tcgen05 phases (7 thread bits): one row per thread in matrix order
                    assert mp[:T] == list(R) + [q for q in range(T) if q not in R], (mp, R)
                    assert ph["op_begin"] == ph["op_end"]
                base = np.zeros(nthreads, dtype=np.int64)
                for k in range(T - rb):
                    base |= ((tid >> k) & 1) << mp[rb + k]
                loc = np.stack([base + sum(1 << mp[i] for i in range(rb) if (rho >> i) & 1)
                                for rho in range(nr)], axis=1)
                v = buf[loc]
                order = list(range(ph["op_begin"], ph["op_mid"])) + ["tc"] + \
                    list(range(ph["op_mid"], ph["op_end"]))
                for o in order:
                    if o == "tc":
                        if ph["tc"] >= 0:
                            U = nat.tc_matrix(p, ph["tc"]).astype(v.dtype)
                            v[:] = v @ U.T
                        continue
                    op = ops[o]
                    if op["kind"] == "perm":  # CNOT on register bits
                        cm, tm = 1 << op["ctrl"], 1 << op["tgt"]
                        for rho in range(nr):
                            if rho & cm and not rho & tm:
                                v[:, [rho, rho | tm]] = v[:, [rho | tm, rho]]
                        continue
                    if op["kind"] == "ctrl":  # U0 / U1 on one register bit, chosen by a thread bit
                        mask = op["mask"]           # or by a shard qubit outside the tile
                        ctb = op["ctrl_thread_bit"]
                        sel = (tid >> ctb) & 1 if ctb >= 0 else np.full(nthreads, int(idx[0] >> (-1 - ctb)) & 1)
                        Us = op["coeffs"].reshape(2, 2, 2).astype(v.dtype)
                        rest = (nr - 1) & ~mask
                        for g in range(1 << (rb - 1)):
                            b0 = _deposit(g, rest, rb)
                            c0, c1 = b0, b0 | mask
                            a0, a1 = v[:, c0].copy(), v[:, c1].copy()
                            v[:, c0] = Us[sel, 0, 0] * a0 + Us[sel, 0, 1] * a1
                            v[:, c1] = Us[sel, 1, 0] * a0 + Us[sel, 1, 1] * a1
                        continue
                    if op["kind"] == "dense":
                        k, mask = op["k"], op["mask"]
                        d = 1 << k
                        M = op["coeffs"].reshape(d, d).astype(v.dtype)
                        rest = (nr - 1) & ~mask
                        for g in range(1 << (rb - k)):
                            b0 = _deposit(g, rest, rb)
                            cols = [b0 | _deposit(j, mask, rb) for j in range(d)]
                            vin = v[:, cols].copy()
                            for i in range(d):
                                v[:, cols[i]] = vin @ M[i]
                    else:
                        kt = op["mask"]
                        kx = len(op["ext_qubits"])
                        kr = op["k"] - kt - kx
                        dt = np.zeros(nthreads, dtype=np.int64)
                        for j, tb in enumerate(op["thread_bits"]):
                            dt |= ((tid >> tb) & 1) << j
                        for j, q in enumerate(op["ext_qubits"]):
                            dt |= (int(idx[0] >> q) & 1) << (kr + kt + j)
                        tab = op["coeffs"].astype(v.dtype)
                        for rho in range(nr):
                            v[:, rho] *= tab[dt | int(op["rmap"][rho])]
                buf[loc] = v
            amps[idx] = buf
    return amps


REG_CASES = [
    ("layered13", lambda: fuse(gen.layered_circuit(13, layers=5, seed=3), 2)[0]),
    ("layered12_w3", lambda: fuse(gen.layered_circuit(12, layers=4, seed=4), 3)[0]),
    ("qft12", lambda: fuse(gen.qft_circuit(12), 2)[0]),
    ("su2_12", lambda: gen.random_su2_circuit(12, 40, seed=9)),
]


@pytest.mark.parametrize("name,make", REG_CASES, ids=[c[0] for c in REG_CASES])
@pytest.mark.parametrize("prec", ["single", "double"])
def test_register_phase_encoding(name, make, prec):
    c = make()
    want = orc.run_circuit(c, "double")
    plan = CircuitPlan(c.num_qubits, Precision(prec), c.gates)
    infos = plan.passes()
    assert all(i["reg_bits"] > 0 and i["num_phases"] >= 1 for i in infos), infos
    got = emulate_reg(plan, c.num_qubits, prec)
    assert np.abs(got - want).max() <= (1e-12 if prec == "double" else 1e-5)


@pytest.mark.parametrize("prec,rb", [("single", 5), ("single", 3), ("double", 4)])
def test_register_phase_encoding_other_widths(prec, rb):
    c = fuse(gen.layered_circuit(14, layers=5, seed=6), 2)[0]
    q = fuse(gen.qft_circuit(13), 2)[0]
    for circ in (c, q):
        want = orc.run_circuit(circ, "double")
        plan = CircuitPlan(circ.num_qubits, Precision(prec), circ.gates,
                           plan_options(reg_bits=rb, tile_bits=rb + 8))
        infos = plan.passes()
        assert all(i["reg_bits"] == rb for i in infos)
        got = emulate_reg(plan, circ.num_qubits, prec)
        assert np.abs(got - want).max() <= (1e-12 if prec == "double" else 1e-5)


@pytest.mark.parametrize("name,make", REG_CASES, ids=[c[0] for c in REG_CASES])
def test_tensor_core_phase_encoding(name, make):
    """k_tc_pass plans (c64): phases whose dense gates fuse into one 32x32
    matrix; emulated with the planner's fused matrices."""
    c = make()
    want = orc.run_circuit(c, "double")
    plan = CircuitPlan(c.num_qubits, Precision.SINGLE, c.gates, plan_options(tensor_cores=1))
    infos = plan.passes()
    assert all(i["tile_bits"] == 12 and i["reg_bits"] == 5 for i in infos)
    got = emulate_reg(plan, c.num_qubits, "single")
    assert np.abs(got - want).max() <= 1e-5
    assert np.abs(plan_order_state(plan, c, "double") - want).max() <= 1e-12


def test_tensor_core_plans_layered28():
    f, _ = fuse(gen.layered_circuit(28), 2)
    plan = CircuitPlan(28, Precision.SINGLE, f.gates, plan_options(tensor_cores=1))
    infos = plan.passes()
    assert sum(i["num_tc"] for i in infos) > 0
    assert len(infos) < 26


@pytest.mark.parametrize("prec", ["single", "double"])
def test_diagonal_gates_outside_the_tile(prec):
    """Diagonal gates need no tile qubits: bits outside the tile are constant
    per tile and select the table entry from the tile origin.  QFT stages then
    share passes (qft-30 c128: 53 passes before, 10 with the parameter-block
    coefficient pool, <= 6 with the c128 pool continued in global memory)."""
    c = fuse(gen.qft_circuit(16), 2)[0]
    want = orc.run_circuit(c, "double")
    plan = CircuitPlan(16, Precision(prec), c.gates)
    infos = plan.passes()
    ext = 0
    for p, info in enumerate(infos):
        for i in range(info["num_kernel_ops"]):
            ext += any(t >= info["tile_bits"] for t in plan.native.kernel_op(p, i)["targets"])
    assert ext > 0
    got = emulate_reg(plan, 16, prec)
    assert np.abs(got - want).max() <= (1e-12 if prec == "double" else 1e-5)
    f30, _ = fuse(gen.qft_circuit(30), 2)
    assert CircuitPlan(30, Precision.DOUBLE, f30.gates).num_passes <= 6


MMA_CASES = [
    ("layered14", lambda: fuse(gen.layered_circuit(14, layers=6, seed=3), 2)[0]),
    ("layered13_w3", lambda: fuse(gen.layered_circuit(13, layers=4, seed=4), 3)[0]),
    ("qft14", lambda: fuse(gen.qft_circuit(14), 2)[0]),
    ("su2_14", lambda: gen.random_su2_circuit(14, 60, seed=9)),
]


@pytest.mark.parametrize("name,make", MMA_CASES, ids=[c[0] for c in MMA_CASES])
def test_mma_phase_encoding(name, make):
    """tensor_cores=2 (c64): whole register phases fused into one 32x32 matrix,
    run by k_reg_pass as an mma.sync GEMM in the fragment layout."""
    c = make()
    want = orc.run_circuit(c, "double")
    plan = CircuitPlan(c.num_qubits, Precision.SINGLE, c.gates, plan_options(tensor_cores=2))
    infos = plan.passes()
    assert all(i["reg_bits"] == 5 for i in infos)
    got = emulate_reg(plan, c.num_qubits, "single")
    assert np.abs(got - want).max() <= 1e-5
    assert np.abs(plan_order_state(plan, c, "double") - want).max() <= 1e-12


def test_mma_plans_layered28():
    f, _ = fuse(gen.layered_circuit(28), 2)
    plan = CircuitPlan(28, Precision.SINGLE, f.gates, plan_options(tensor_cores=2))
    infos = plan.passes()
    assert sum(i["num_tc"] for i in infos) > 0
    assert sum(i["num_gates"] for i in infos) == 189


def _mixed_circuit(n: int, layers: int, seed: int) -> Circuit:
    """Dense 2q gates on neighbours, diagonal CP / CZ-type gates on far pairs,
    RZ and H: fused passes whose GEMMs interleave with diagonal ops on row and
    outside-tile qubits."""
    rng = np.random.default_rng(seed)
    gates = []
    for layer in range(layers):
        for q in range(layer % 2, n - 1, 2):
            z = rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4))
            u, _ = np.linalg.qr(z)
            gates.append(GateOp(GateKind.CUSTOM, (q, q + 1), (), u))
        for _ in range(n // 2):
            a, b = (int(x) for x in rng.choice(n, 2, replace=False))
            ph = np.exp(1j * rng.uniform(0, 2 * np.pi, 4))
            gates.append(GateOp(GateKind.CUSTOM, (min(a, b), max(a, b)), (), np.diag(ph)))
        for q in range(n):
            gates.append(GateOp(GateKind.RZ if (q + layer) % 3 else GateKind.H, (q,),
                                (rng.uniform(0, 6),) if (q + layer) % 3 else ()))
    return Circuit(n, gates)


GEMM_CASES = [
    ("layered16", lambda: fuse(gen.layered_circuit(16, layers=8, seed=2), 2)[0]),
    ("qft16", lambda: fuse(gen.qft_circuit(16), 2)[0]),
    ("qft18_w3", lambda: fuse(gen.qft_circuit(18), 3)[0]),
    ("mixed15", lambda: fuse(_mixed_circuit(15, 6, 3), 2)[0]),
    ("mixed14_raw", lambda: _mixed_circuit(14, 4, 4)),
]


@pytest.mark.parametrize("name,make", GEMM_CASES, ids=[c[0] for c in GEMM_CASES])
def test_gemm_pass_encoding(name, make):
    """k_gemm_pass lowering (c64 default): load layout, GEMMs on the column
    qubits in matrix order, diagonal ops moved across / between GEMMs, 32x32b
    and 16x256b read-out layouts -- emulated against the oracle."""
    c = make()
    want = orc.run_circuit(c, "double")
    plan = CircuitPlan(c.num_qubits, Precision.SINGLE, c.gates)
    infos = plan.passes()
    gemm = [i for i in infos if i["kernel"] == "gemm"]
    assert gemm, infos
    got = emulate_reg(plan, c.num_qubits, "single")
    assert np.abs(got - want).max() <= 1e-5
    assert np.abs(plan_order_state(plan, c, "double") - want).max() <= 1e-12


def test_gemm_plans_cover_diagonals_and_readouts():
    layouts = set()
    with_ops = 0
    for _name, make in GEMM_CASES:
        c = make()
        plan = CircuitPlan(c.num_qubits, Precision.SINGLE, c.gates)
        nat = plan.native
        for p, info in enumerate(plan.passes()):
            if info["kernel"] != "gemm":
                continue
            with_ops += info["num_kernel_ops"] > 0
            for f in range(info["num_phases"]):
                layouts.add(bool(nat.phase(p, f)["flags"] & 8))
    assert with_ops > 0 and layouts == {False, True}


FACTOR_CASES = [
    ("layered14", lambda: fuse(gen.layered_circuit(14, layers=6, seed=3), 2)[0]),
    ("layered13_w2b", lambda: fuse(gen.layered_circuit(13, layers=8, seed=8), 2)[0]),
    ("qft13", lambda: fuse(gen.qft_circuit(13), 2)[0]),
    ("mixed14", lambda: fuse(_mixed_circuit(14, 4, 6), 2)[0]),
]


@pytest.mark.parametrize("name,make", FACTOR_CASES, ids=[c[0] for c in FACTOR_CASES])
def test_c128_factorised_gates(name, make):
    """c128 plans factor fused 2q gates as D P (A x B) (1-qubit ops with real /
    imaginary columns, a CNOT register permutation, the diagonal merged into a
    run): register-phase and shared-memory lowering both emulated."""
    c = make()
    want = orc.run_circuit(c, "double")
    plan = CircuitPlan(c.num_qubits, Precision.DOUBLE, c.gates, plan_options(no_factor=-1))
    kinds = [plan.native.kernel_op(p, i)["kind"] for p in range(plan.num_passes)
             for i in range(plan.native.pass_info(p)["num_kernel_ops"])]
    if name.startswith("layered"):
        assert "perm" in kinds
    assert np.abs(emulate_reg(plan, c.num_qubits, "double") - want).max() <= 1e-12
    assert np.abs(plan_order_state(plan, c, "double") - want).max() <= 1e-12
    tile = CircuitPlan(c.num_qubits, Precision.DOUBLE, c.gates, plan_options(no_reg_phases=1, no_factor=-1))
    assert np.abs(emulate(tile, c.num_qubits, "double") - want).max() <= 1e-12
    plain = CircuitPlan(c.num_qubits, Precision.DOUBLE, c.gates)  # default: dense
    assert all(plain.native.kernel_op(p, i)["kind"] != "perm" for p in range(plain.num_passes)
               for i in range(plain.native.pass_info(p)["num_kernel_ops"]))


def test_gate_merge_of_unfused_runs():
    """Unfused input (the paper's Table-2 circuits): runs of dense gates on the
    same qubits become one op; pass_gates still lists every input gate, and
    the state equals the oracle's and the unmerged plan's."""
    c = gen.random_su2_circuit(10, 100, seed=3)
    want = orc.run_circuit(c, "double")
    o = dict(tensor_cores=-1, tile_bits=8, min_low_bits=2)
    merged = CircuitPlan(10, Precision.DOUBLE, c.gates, plan_options(**o))
    plain = CircuitPlan(10, Precision.DOUBLE, c.gates, plan_options(no_gate_merge=1, **o))
    n_ops = [sum(p.native.pass_info(i)["num_kernel_ops"] for i in range(p.num_passes)) for p in (merged, plain)]
    assert n_ops[0] < n_ops[1] and n_ops[1] >= 100
    assert sum(i["num_gates"] for i in merged.passes()) == len(c.gates)
    for p in (merged, plain):
        assert np.abs(plan_order_state(p, c, "double") - want).max() <= 1e-12
        assert np.abs(emulate(p, 10, "double") - want).max() <= 1e-12
    # a 2q gate absorbs the open 1q gates on its qubits; a diagonal gate blocks a merge
    g = [GateOp(GateKind.H, (0,)), GateOp(GateKind.RX, (1,), (0.3,)), GateOp(GateKind.CNOT, (0, 1)),
         GateOp(GateKind.RZ, (1,), (0.7,)), GateOp(GateKind.RY, (1,), (0.2,)), GateOp(GateKind.H, (0,))]
    c2 = Circuit(4, g)
    p2 = CircuitPlan(4, Precision.DOUBLE, g, plan_options(tensor_cores=-1, tile_bits=4, min_low_bits=1))
    assert np.abs(emulate(p2, 4, "double") - orc.run_circuit(c2, "double")).max() <= 1e-12
    assert sum(i["num_kernel_ops"] for i in p2.passes()) < len(g)


def test_controlled_ops_on_thread_bits():
    """Block-diagonal (controlled-U) 2q gates whose control is not a register
    bit of the phase run as OP_CTRL (U0 / U1 selected by a thread bit): the
    c128 layered and QFT plans use them, and the register-phase emulation with
    them reproduces the oracle."""
    for c in (fuse(gen.layered_circuit(13, layers=5, seed=3), 2)[0], fuse(gen.qft_circuit(12), 2)[0]):
        plan = CircuitPlan(c.num_qubits, Precision.DOUBLE, c.gates)
        infos = plan.passes()
        kinds = [plan.native.phase_op(p, k)["kind"] for p in range(plan.num_passes)
                 for k in range(infos[p]["num_kernel_ops"])]
        assert "ctrl" in kinds
        got = emulate_reg(plan, c.num_qubits, "double")
        assert np.abs(got - orc.run_circuit(c, "double")).max() <= 1e-12


def test_controls_outside_the_tile():
    """c128: a controlled 2q gate needs only its target in the tile; with the
    control outside, the pass applies U0 / U1 per tile (kernel op "ctrl",
    phase op with a negative control thread bit).  Both emulations (tile
    kernel view and register phases) reproduce the oracle, and switching the
    feature off (SVB_NO_CTRLX) costs passes on a layered circuit."""
    import os
    c = fuse(gen.layered_circuit(16, layers=8, seed=5), 2)[0]
    plan = CircuitPlan(16, Precision.DOUBLE, c.gates)
    infos = plan.passes()
    kops = [plan.native.kernel_op(p, k) for p in range(plan.num_passes) for k in range(infos[p]["num_kernel_ops"])]
    assert any(o["kind"] == "ctrl" for o in kops)
    want = orc.run_circuit(c, "double")
    assert np.abs(plan_order_state(plan, c, "double") - want).max() <= 1e-12
    assert np.abs(emulate_reg(plan, 16, "double") - want).max() <= 1e-12
    os.environ["SVB_NO_CTRLX"] = "1"
    try:
        plain = CircuitPlan(16, Precision.DOUBLE, c.gates)
    finally:
        del os.environ["SVB_NO_CTRLX"]
    assert plan.num_passes <= plain.num_passes


def test_c128_pool_past_the_parameter_block():
    """c128 passes may hold a 64 KB coefficient pool (kPoolBytesC128): the
    part past the 24 KB kernel-parameter block lives in global memory.  QFT
    passes fill it with merged diagonal tables; c64 passes stay within 24 KB.
    (The GPU QFT tests on random states run these plans against the oracle.)"""
    param_elems = {"double": 24576 // 16, "single": 24576 // 8}
    cap_elems = {"double": 65536 // 16, "single": 24576 // 8}
    f16, _ = fuse(gen.qft_circuit(16), 2)
    big = {}
    for prec in ("double", "single"):
        plan = CircuitPlan(16, Precision(prec), f16.gates)
        pools = [sum(len(plan.native.kernel_op(p, i)["coeffs"])
                     for i in range(plan.native.pass_info(p)["num_kernel_ops"]))
                 for p in range(plan.num_passes)]
        assert max(pools) <= cap_elems[prec]
        big[prec] = max(pools) > param_elems[prec]
    assert big["double"] and not big["single"]
