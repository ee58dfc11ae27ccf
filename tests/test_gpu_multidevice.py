"""Sharding behind the Engine plugin API (paper_2604_03816_b200.multidevice).

On a one-GPU box the shards are placed on the same device (``devices=[0]``,
``shards=P``): every code path -- sharded |0>, localised diagonal gates on
global qubits, block exchanges between shards, the per-gate (checkpoint) path,
layout canonicalisation, chunked host views, shard-by-shard sampling, inner
products -- runs exactly as it would over P GPUs, with peer copies replaced by
same-device copies.  Tolerances are the north star's.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import has_cuda
from oracle import sv_oracle as orc
from paper_2604_03816_b200 import generators as gen
from paper_2604_03816_b200.b200 import B200Engine
from paper_2604_03816_b200.circuit import Circuit, GateKind, GateOp, Precision
from paper_2604_03816_b200.engines import AllocationError
from paper_2604_03816_b200.fusion import fuse
from paper_2604_03816_b200.multidevice import ShardedDeviceState

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")]

TOL = {"double": 1e-12, "single": 1e-5}


def check(got, want, prec):
    err = float(np.abs(got.astype(np.complex128) - want.astype(np.complex128)).max())
    assert err <= TOL[prec], err
    assert orc.normalised_fidelity(got, want) >= 1 - (1e-10 if prec == "double" else 1e-5)


CIRCS = {
    "layered16": lambda: fuse(gen.layered_circuit(16, layers=8, seed=3), 2)[0],
    "qft15": lambda: fuse(gen.qft_circuit(15), 2)[0],
    "su2_14": lambda: gen.random_su2_circuit(14, 80, seed=4),
}


@pytest.mark.parametrize("name", list(CIRCS))
@pytest.mark.parametrize("shards", [2, 4, 8])
@pytest.mark.parametrize("prec", ["double", "single"])
def test_sharded_run_circuit_vs_oracle(name, shards, prec):
    c = CIRCS[name]()
    eng = B200Engine("b200-md", devices=[0], shards=shards)
    st = eng.run_circuit(c, Precision(prec))
    assert isinstance(st, ShardedDeviceState) and st.world == shards
    want = orc.run_circuit(c, prec)
    check(st.amplitudes, want, prec)
    assert abs(st.norm_squared() - 1) <= (1e-10 if prec == "double" else 1e-5)
    eng.release(st)
    assert eng.live_states == 0


def test_sharded_checkpoint_path_and_adopt():
    """Per-gate path on a sharded state (the checkpoint hook, ref
    engines.py:174-187) and adopt of a random host state."""
    c = fuse(gen.layered_circuit(13, layers=4, seed=5), 2)[0]
    eng = B200Engine("b200-md-cp", devices=[0], shards=4)
    seen = []
    st = eng.run_circuit(c, Precision.DOUBLE, checkpoint=lambda s, i: seen.append(i))
    assert seen == list(range(len(c.gates)))
    check(st.amplitudes, orc.run_circuit(c, "double"), "double")
    eng.release(st)
    rng = np.random.default_rng(2)
    init = rng.normal(size=1 << 13) + 1j * rng.normal(size=1 << 13)
    init /= np.linalg.norm(init)
    st = eng.adopt(13, Precision.DOUBLE, init)
    for op in c.gates:
        eng.apply_gate(st, op)
    want = init.copy()
    for op in c.gates:
        orc.apply_gate(want, 13, op)
    check(st.amplitudes, want, "double")
    eng.release(st)
    assert eng.live_states == 0


def test_sharded_sampling_and_inner_products():
    def ref_sample(amps, shots, seed, n):
        probs = np.abs(amps.astype(np.complex128)) ** 2
        cdf = np.cumsum(probs)
        draws = np.random.Generator(np.random.Philox(key=seed)).random(shots)
        idx = np.minimum(np.searchsorted(cdf, draws * cdf[-1], side="right"), len(cdf) - 1)
        v, cnt = np.unique(idx, return_counts=True)
        return {format(int(a), f"0{n}b"): int(b) for a, b in zip(v, cnt)}
    eng = B200Engine("b200-md-s", devices=[0], shards=4)
    for circ in (gen.ghz_circuit(12), fuse(gen.qft_circuit(14), 2)[0],
                 fuse(gen.layered_circuit(14, layers=5, seed=1), 2)[0]):
        st = eng.run_circuit(circ, Precision.DOUBLE)
        got = eng.sample(st, 4096, seed=7)
        assert got.counts == ref_sample(st.amplitudes, 4096, 7, circ.num_qubits)
        assert np.abs(eng.probabilities(st) - np.abs(st.amplitudes) ** 2).max() <= 1e-15
        eng.release(st)
    a = eng.run_circuit(fuse(gen.layered_circuit(14, layers=5, seed=1), 2)[0], Precision.DOUBLE)
    b = eng.run_circuit(fuse(gen.qft_circuit(14), 2)[0], Precision.DOUBLE)
    assert abs(eng.inner(a, b) - np.vdot(a.amplitudes, b.amplitudes)) <= 1e-12
    assert abs(eng.fidelity(a, a) - 1) <= 1e-12


def test_allocation_error_when_no_device_set_fits():
    eng = B200Engine("b200-all", devices="all")
    with pytest.raises(AllocationError):
        eng.init_state(42, Precision.DOUBLE)  # 64 TiB
    assert eng.live_states == 0


def test_sharded_30q_c64_matches_single_device():
    """A 30-qubit c64 layered circuit on 2 shards (8 GiB blocks exchanged)
    equals the single-device result."""
    import torch
    f, _ = fuse(gen.layered_circuit(30, layers=6, seed=9), 2)
    one = B200Engine("b200-one")
    ref = one.run_circuit(f, Precision.SINGLE)
    eng = B200Engine("b200-md30", devices=[0], shards=2)
    st = eng.run_circuit(f, Precision.SINGLE)
    from paper_2604_03816_b200.multidevice import canonicalize
    canonicalize(st)
    half = 1 << 29
    for r, sh in enumerate(st.shards):
        d = (sh.tensor - ref.tensor[r * half:(r + 1) * half]).abs().max().item()
        assert d <= 1e-5, d
    assert abs(st.norm_squared() - 1) <= 1e-5
    eng.release(st)
    one.release(ref)
    del st, ref
    torch.cuda.empty_cache()
