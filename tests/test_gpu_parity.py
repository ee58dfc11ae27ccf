"""GPU parity: the CUDA engine (through libsvb200.so) against the CPU oracle.

Tolerances (BASELINE.json north_star): complex128 max-abs <= 1e-12 and
fidelity >= 1 - 1e-10; complex64 max-abs <= 1e-5 and fidelity >= 1 - 1e-5,
fidelity normalised as SURVEY.md 8(a14) explains (the reference's own c64
norm drift would otherwise consume the budget).  At sizes the oracle cannot
reach, size-independent properties are used: QFT|0> is exactly uniform,
mirror circuits C^dagger C return |0>, norms are preserved.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import has_cuda
from golden_io import decode
from oracle import sv_oracle as orc
from paper_2604_03816_b200 import generators as gen
from paper_2604_03816_b200.b200 import B200Engine, plan_options
from paper_2604_03816_b200.circuit import Circuit, GateKind, GateOp, Precision, effective_unitary
from paper_2604_03816_b200.engines import AllocationError
from paper_2604_03816_b200.fusion import fuse

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")]

TOL = {"double": (1e-12, 1e-10), "single": (1e-5, 1e-5)}


@pytest.fixture(scope="module")
def eng():
    return B200Engine("b200-test")


def assert_close(got: np.ndarray, want: np.ndarray, prec: str, what=""):
    amax, ftol = TOL[prec]
    err = float(np.abs(got.astype(np.complex128) - want.astype(np.complex128)).max())
    fid = orc.normalised_fidelity(got, want)
    assert err <= amax, f"{what} max-abs {err:.3e} > {amax}"
    assert fid >= 1 - ftol, f"{what} fidelity 1-{1 - fid:.3e}"


def test_known_answers(eng):
    inv = 1 / math.sqrt(2)
    s = eng.run_circuit(Circuit(2, [GateOp(GateKind.H, (0,))]))
    assert np.allclose(s.amplitudes, [inv, inv, 0, 0], atol=1e-15)
    s = eng.run_circuit(gen.ghz_circuit(2))
    assert np.allclose(s.amplitudes, [inv, 0, 0, inv], atol=1e-15)
    for n in (1, 2, 3, 5, 13, 14):
        for t in range(n):
            s = eng.run_circuit(Circuit(n, [GateOp(GateKind.X, (t,))]))
            e = np.zeros(1 << n)
            e[1 << t] = 1
            assert np.array_equal(s.amplitudes, e), (n, t)
    s = eng.run_circuit(gen.ghz_circuit(5))
    e = np.zeros(32, dtype=complex)
    e[0] = e[31] = inv
    assert np.allclose(s.amplitudes, e, atol=1e-15)
    s = eng.run_circuit(Circuit(3, []))
    assert np.array_equal(s.amplitudes, [1, 0, 0, 0, 0, 0, 0, 0])


@pytest.mark.parametrize("prec", ["double", "single"])
def test_golden_random_circuits(eng, golden_random, prec):
    key = "c128" if prec == "double" else "c64"
    for i in range(int(golden_random["count"])):
        c = decode(f"c{i}_", golden_random)
        want = golden_random[f"c{i}_{key}"]
        planned = eng.run_circuit(c, Precision(prec))
        assert planned.amplitudes.dtype == want.dtype
        assert_close(planned.amplitudes, want, prec, f"plan c{i}")
        per_gate = eng.run_circuit(c, Precision(prec), checkpoint=lambda s, j: None)
        assert_close(per_gate.amplitudes, want, prec, f"per-gate c{i}")


@pytest.mark.parametrize("prec", ["double", "single"])
def test_golden_fused_circuits(eng, golden_fused, prec):
    key = "c128" if prec == "double" else "c64"
    for name in golden_fused["names"]:
        c = decode(f"{name}_fused_", golden_fused)
        assert_close(eng.run_circuit(c, Precision(prec)).amplitudes,
                     golden_fused[f"{name}_{key}"], prec, name)


OPTS = [{}, {"tile_bits": 6, "min_low_bits": 2}, {"tile_bits": 9, "min_low_bits": 1, "cost_budget": -1.0},
        {"no_diag_merge": 1, "stages": 2}, {"stages": 4, "max_ops_per_pass": 1},
        {"no_reg_phases": 1}, {"reg_bits": 3, "tile_bits": 11}, {"cost_budget": -1.0, "stages": 2},
        {"reg_bits": 5, "tile_bits": 13, "cost_budget": 3.0, "tensor_cores": -1},
        {"cost_budget": 6.0}, {"tensor_cores": -1, "no_window_search": 1},
        {"tensor_cores": 2}, {"tensor_cores": 2, "tc_min_dense": 1, "cost_budget": 20.0},
        {"tile_bits": 12}, {"tile_bits": 12, "stages": 2, "tensor_cores": -1},
        {"tile_bits": 13}, {"tile_bits": 13, "tc_min_dense": 1}, {"streams": 2}, {"streams": 1}, {"streams": 3}, {"streams": 4}, {"streams": 2, "tile_bits": 12},
        {"no_factor": -1}, {"gemm_warps": 8}, {"tensor_cores": 2}]


@pytest.mark.parametrize("opts", OPTS, ids=[str(o) for o in OPTS])
@pytest.mark.parametrize("prec", ["double", "single"])
def test_plan_shapes_vs_oracle(prec, opts):
    e = B200Engine("b200-opts", options=plan_options(**opts) if opts else None)
    for c in (fuse(gen.layered_circuit(14, layers=6, seed=1), 2)[0],
              fuse(gen.layered_circuit(16, layers=8, seed=2), 2)[0],
              fuse(gen.qft_circuit(13), 2)[0],
              fuse(gen.layered_circuit(13, layers=4, seed=5), 3)[0],
              gen.random_su2_circuit(15, 90, seed=3)):
        want = orc.run_circuit(c, prec)
        assert_close(e.run_circuit(c, Precision(prec)).amplitudes, want, prec, c.name)


@pytest.mark.parametrize("prec", ["double", "single"])
def test_every_target_and_pair(eng, prec):
    rng = np.random.default_rng(7)
    n = 15
    for t in range(n):
        u = orc.gate_unitary(GateOp(GateKind.U3, (t,), tuple(rng.uniform(0, 6, 3))))
        c = Circuit(n, [GateOp(GateKind.H, (q,)) for q in range(n)] +
                    [GateOp(GateKind.CUSTOM, (t,), (), u)])
        assert_close(eng.run_circuit(c, Precision(prec)).amplitudes, orc.run_circuit(c, prec), prec)
    for _ in range(12):
        a, b = (int(x) for x in rng.choice(n, 2, replace=False))
        z = rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4))
        q, _ = np.linalg.qr(z)
        c = Circuit(n, [GateOp(GateKind.RY, (x,), (0.3 * x + 0.1,)) for x in range(n)] +
                    [GateOp(GateKind.CUSTOM, (a, b), (), q)])
        assert_close(eng.run_circuit(c, Precision(prec)).amplitudes, orc.run_circuit(c, prec), prec)


@pytest.mark.parametrize("prec", ["double", "single"])
def test_qft18_outside_tile_diagonals(eng, prec):
    """QFT at 18 q: multi-pass plans whose merged diagonal tables read shard
    qubits outside the tile (per-tile index parts), and fused CP runs."""
    f, _ = fuse(gen.qft_circuit(18), 2)
    plan = eng.plan(f, Precision(prec))
    ext = 0
    for p in range(plan.num_passes):
        info = plan.native.pass_info(p)
        for i in range(info["num_kernel_ops"]):
            ext += any(t >= info["tile_bits"] for t in plan.native.kernel_op(p, i)["targets"])
    assert plan.num_passes >= 2 and ext > 0
    assert_close(eng.run_circuit(f, Precision(prec)).amplitudes, orc.run_circuit(f, prec), prec, "qft18")
    raw = gen.qft_circuit(16)  # unfused: 1q RZ / CNOT / H stream
    assert_close(eng.run_circuit(raw, Precision(prec)).amplitudes, orc.run_circuit(raw, prec), prec, "qft16 raw")


@pytest.mark.parametrize("prec", ["double", "single"])
def test_non_unitary_and_unnormalised(eng, prec):
    """CUSTOM matrices need not be unitary and adopted states need not be
    normalised (the reference applies whatever it is given): the tensor-core
    phases' per-row scaling adapts to any magnitude and passes with a
    non-unitary op skip the norm restoration."""
    rng = np.random.default_rng(21)
    n = 15
    gates = []
    for layer in range(6):
        for q in range(layer % 2, n - 1, 2):
            m = rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4))
            if (layer + q) % 3:
                m, _ = np.linalg.qr(m)
            else:
                m = 0.7 * m  # non-unitary
            gates.append(GateOp(GateKind.CUSTOM, (q, q + 1), (), m))
    c = Circuit(n, gates)
    init = (rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)) * 3.0
    init = init.astype(np.complex128 if prec == "double" else np.complex64)
    st = eng.adopt(n, Precision(prec), init.copy())
    for op in c.gates:  # per-gate path
        eng.apply_gate(st, op)
    want = init.copy()
    for op in c.gates:
        orc.apply_gate(want, n, op)
    got = st.amplitudes
    scale = float(np.abs(want).max())
    err = float(np.abs(got.astype(np.complex128) - want.astype(np.complex128)).max()) / scale
    assert err <= (1e-12 if prec == "double" else 1e-5), err
    eng.release(st)
    # the planned path (fused phases, tensor cores for c64) from the same state
    plan = eng.plan(c, Precision(prec))
    st = eng.adopt(n, Precision(prec), init.copy())
    eng.execute(st, plan)
    got = st.amplitudes
    err = float(np.abs(got.astype(np.complex128) - want.astype(np.complex128)).max()) / scale
    assert err <= (1e-12 if prec == "double" else 1e-5), err
    eng.release(st)


def test_layered20_config1_vs_oracle(eng):
    """BASELINE config 1 workload (layered-20, c128, fused 693 -> 133)."""
    f, rep = fuse(gen.layered_circuit(20), 2)
    assert (rep.original_gate_count, rep.fused_gate_count) == (693, 133)
    want = orc.run_circuit(f, "double")
    assert_close(eng.run_circuit(f, Precision.DOUBLE).amplitudes, want, "double", "layered-20")
    want1 = orc.run_circuit(f, "single")
    assert_close(eng.run_circuit(f, Precision.SINGLE).amplitudes, want1, "single", "layered-20 c64")


def test_qft30_c128_uniform(eng):
    """BASELINE config 3 at full size: QFT|0...0> is exactly uniform (2^-15)."""
    import torch
    f, _ = fuse(gen.qft_circuit(30), 2)
    s = eng.run_circuit(f, Precision.DOUBLE)
    dev = s.tensor
    # the CP decomposition (ref generators.py:37-45) is exact up to a global
    # phase, so the output is a0 * (1, ..., 1) with |a0| = 2^-15
    a0 = dev[0].item()
    assert abs(abs(a0) - 2.0 ** -15) <= 1e-12
    err = float((dev - a0).abs().max().item())
    assert err <= 1e-12, err
    assert abs(eng.norm_squared(s) - 1.0) <= 1e-10
    eng.release(s)
    del dev
    torch.cuda.empty_cache()


def _dagger(c):
    return Circuit(c.num_qubits, [GateOp(GateKind.CUSTOM, op.targets, (),
                                         effective_unitary(op).conj().T) for op in reversed(c.gates)])


def test_mirror28_c64(eng):
    """BASELINE config 2 shape: layered-28 c64, then its inverse -> |0>."""
    import torch
    f, _ = fuse(gen.layered_circuit(28), 2)
    mirror = Circuit(28, list(f.gates) + list(_dagger(f).gates))
    s = eng.run_circuit(mirror, Precision.SINGLE)
    a0 = complex(s.tensor[0].item())
    assert abs(abs(a0) - 1.0) <= 1e-5
    assert abs(eng.norm_squared(s) - 1.0) <= 1e-5
    eng.release(s)
    torch.cuda.empty_cache()


def test_reductions(eng):
    f, _ = fuse(gen.layered_circuit(16, layers=3), 2)
    a = eng.run_circuit(f, Precision.DOUBLE)
    b = eng.run_circuit(gen.qft_circuit(16), Precision.DOUBLE)
    ha, hb = a.amplitudes, b.amplitudes
    assert abs(eng.inner(a, b) - np.vdot(ha, hb)) <= 1e-12
    assert abs(eng.norm_squared(a) - np.vdot(ha, ha).real) <= 1e-12
    assert np.abs(eng.probabilities(a) - np.abs(ha) ** 2).max() <= 1e-15
    a1 = eng.run_circuit(f, Precision.SINGLE)
    assert abs(eng.fidelity(a, a1, normalised=True) - 1) <= 1e-6


def test_engine_api_contract():
    e = B200Engine("b200-api", capacity_bytes=16 << 30)
    with pytest.raises(AllocationError) as ei:
        e.init_state(30, Precision.DOUBLE)
    assert ei.value.requested_bytes == 17_179_869_184
    assert e.live_states == 0
    s = e.init_state(3, Precision.SINGLE)
    assert e.live_states == 1
    assert s.amplitudes.dtype == np.complex64
    with pytest.raises(ValueError):
        e.apply_gate(s, GateOp(GateKind.X, (3,)))
    e.release(s)
    assert e.live_states == 0
    with pytest.raises(ValueError):
        e.init_state(0, Precision.DOUBLE)
    host = np.zeros(8, dtype=np.complex128)
    host[5] = 1
    s = e.adopt(3, Precision.DOUBLE, host)
    e.apply_gate(s, GateOp(GateKind.X, (0,)))
    assert s.amplitudes[4] == 1
    e.release(s)


def test_device_sampling_matches_reference_semantics(eng):
    """sample() keeps ref engines.py:307-337 semantics: same counts as the
    numpy inverse-CDF path on the same probabilities and Philox seed."""
    def ref_sample(amps, shots, seed, n):
        probs = np.abs(amps.astype(np.complex128)) ** 2
        cdf = np.cumsum(probs)
        draws = np.random.Generator(np.random.Philox(key=seed)).random(shots)
        idx = np.minimum(np.searchsorted(cdf, draws * cdf[-1], side="right"), len(cdf) - 1)
        v, c = np.unique(idx, return_counts=True)
        return {format(int(a), f"0{n}b"): int(b) for a, b in zip(v, c)}
    for n, circ in ((4, gen.ghz_circuit(4)), (10, fuse(gen.layered_circuit(10, layers=3), 2)[0]),
                    (14, gen.qft_circuit(14))):
        for prec in (Precision.DOUBLE, Precision.SINGLE):
            s = eng.run_circuit(circ, prec)
            got = eng.sample(s, 4096, seed=11)
            assert got.shots == 4096 and sum(got.counts.values()) == 4096
            assert got.counts == ref_sample(s.amplitudes, 4096, 11, n)
    s = eng.run_circuit(gen.ghz_circuit(4), Precision.DOUBLE)
    assert eng.sample(s, 0, seed=1).counts == {}


def test_layered33_c128_mirror_full_size(eng):
    """BASELINE config 4 at full size (33 q, complex128, 128 GiB state): the
    fused layered circuit followed by its inverse returns |0...0>."""
    import torch
    free, _ = torch.cuda.mem_get_info()
    if free < (1 << 37) + (8 << 30):
        pytest.skip("needs ~136 GiB free device memory")
    f, rep = fuse(gen.layered_circuit(33), 2)
    assert rep.fused_gate_count == 224
    mirror = Circuit(33, list(f.gates) + list(_dagger(f).gates))
    s = eng.run_circuit(mirror, Precision.DOUBLE)
    a0 = complex(s.tensor[0].item())
    assert abs(a0 - 1.0) <= 1e-10, a0
    assert abs(eng.norm_squared(s) - 1.0) <= 1e-10
    eng.release(s)
    del s
    torch.cuda.empty_cache()


def test_reference_registry_dropin():
    """With the reference package importable (baseline/_ref travels to the GPU
    box; tests/conftest.py appends it), ``aqsim.run_circuit("b200")`` runs on
    the device and matches the reference engine."""
    aqsim = pytest.importorskip("aqsim")
    import paper_2604_03816_b200  # noqa: F401  (registers "b200")
    c = aqsim.qft_circuit(8)
    got = aqsim.run_circuit("b200", c, aqsim.Precision.DOUBLE)
    want = aqsim.run_circuit("reference", c, aqsim.Precision.DOUBLE)
    assert np.abs(got.amplitudes - want.amplitudes).max() <= 1e-12
    assert aqsim.state_fidelity(got, want) == pytest.approx(1.0, abs=1e-10)


def test_reference_selector_profiles_the_device_engine():
    """aqsim's own selector (ref selector.py:93-118, 127-170) benchmarks every
    available engine through the plugin API -- init_state / apply_gate /
    synchronize / release -- and here that includes the device engine."""
    aqsim = pytest.importorskip("aqsim")
    from aqsim import selector
    import paper_2604_03816_b200  # noqa: F401  (registers "b200")
    engines = aqsim.registered_engines()
    assert "b200" in {e.name for e in engines}
    choice, profiles = selector.select(aqsim.ghz_circuit(16), engines)
    prof = {p.engine.name: p for p in profiles}
    assert "b200" in prof and prof["b200"].throughput > 0
    assert choice.name in prof


def test_cli_run_and_bench_scaling(capsys):
    import json as _json
    from paper_2604_03816_b200.__main__ import main
    assert main(["run", "ghz-5", "--shots", "1000", "--seed", "3", "--no-timing"]) == 0
    rep = _json.loads(capsys.readouterr().out)
    assert rep["engine_chosen"] == "b200" and rep["g_fused"] >= 1
    assert set(rep["counts"]) == {"00000", "11111"} and sum(rep["counts"].values()) == 1000
    assert main(["bench-scaling", "--qubits", "10,12", "--repetitions", "1", "--no-timing"]) == 0
    rows = _json.loads(capsys.readouterr().out)
    assert [r["n"] for r in rows] == [10, 12]
    assert main(["bench-fusion", "--circuits", "qft-10", "--repetitions", "1"]) == 0
    rows = _json.loads(capsys.readouterr().out)
    assert rows[0]["fused_time_s"] > 0


def _sharded_cuda_worker(rank, world, port, out, p2p=False):
    """One rank of the sharded engine on cuda:0 with its CUDA local plans;
    exchanges over gloo through host memory (one GPU on this box), or with
    p2p the swap kernel on CUDA-IPC-mapped peer shards (gloo only carries the
    handles and the barriers)."""
    import os
    import torch.distributed as dist
    from paper_2604_03816_b200.sharded import CudaShardBackend, ShardedEngine
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        errs = []
        for c, prec in ((fuse(gen.layered_circuit(16, layers=6, seed=4), 2)[0], "single"),
                        (fuse(gen.qft_circuit(15), 2)[0], "double")):
            eng = ShardedEngine(CudaShardBackend(0), p2p=p2p)
            st = eng.run_circuit(c, Precision(prec))
            full = st.gather()
            norm = st.norm_squared()
            if rank == 0:
                want = orc.run_circuit(c, prec)
                errs += [float(np.abs(full.astype(np.complex128) - want.astype(np.complex128)).max()),
                         abs(norm - 1), st.schedule.num_swaps()]
            if p2p:
                errs.append(float(len(eng._bases)))  # peer shards were IPC-mapped
            eng.close()
        if rank == 0:
            np.save(out, np.array(errs))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,p2p", [(2, False), (4, False), (2, True), (4, True)])
def test_sharded_engine_on_device(world, p2p):
    """The multi-GPU engine end to end with the CUDA backend: `world` ranks
    share cuda:0, local segments run the native plans (including diagonal
    gates restricted to each rank's global bits), swaps over gloo."""
    import os
    import socket
    import tempfile
    import torch.multiprocessing as mp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "res.npy")
        mp.spawn(_sharded_cuda_worker, args=(world, port, out, p2p), nprocs=world, join=True)
        res = np.load(out)
    if p2p:
        e64, n64, s64, m64, e128, n128, s128, m128 = res
        assert m64 == world - 1 and m128 == world - 1
    else:
        e64, n64, s64, e128, n128, s128 = res
    assert e64 <= 1e-5 and n64 <= 1e-5 and s64 >= 1
    assert e128 <= 1e-12 and n128 <= 1e-10 and s128 >= 1
