"""The fusion mirror (``paper_2604_03816_b200.fusion``) against the reference
pass ``aqsim.dag.fuse`` (ref pkg/src/aqsim/dag.py:177-217).

``tests/golden/make_golden.py`` ran the REAL reference fusion on six circuits
(layered, QFT, SU(2), GHZ at widths 2 and 3) and stored input and output op
lists in ``fused_circuits.npz``; it also stored the fused gate counts and
depths at the BASELINE configs in ``fusion_stats.json``.  The mirror must
reproduce both exactly: same op order, kinds, targets, and bit-identical
complex128 matrices (the planner lowers whatever ``fuse`` emits, so any
deviation would change every downstream plan).
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

from golden_io import decode
from paper_2604_03816_b200 import generators as gen
from paper_2604_03816_b200.circuit import GateKind, effective_unitary
from paper_2604_03816_b200.fusion import depth, fuse

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def fused_golden():
    return np.load(os.path.join(GOLDEN, "fused_circuits.npz"))


def test_fuse_matches_reference_op_lists(fused_golden):
    z = fused_golden
    for name in z["names"]:
        orig = decode(f"{name}_orig_", z)
        want = decode(f"{name}_fused_", z)
        width = int(z[f"{name}_width"])
        got, rep = fuse(orig, width)
        assert rep.original_gate_count == len(orig.gates), name
        assert rep.fused_gate_count == len(want.gates) == len(got.gates), name
        for i, (a, b) in enumerate(zip(got.gates, want.gates)):
            assert a.kind == b.kind, (name, i, a.kind, b.kind)
            assert tuple(a.targets) == tuple(b.targets), (name, i)
            if b.kind is GateKind.CUSTOM:
                # bit-identical: same merge order, same complex128 products
                assert np.array_equal(effective_unitary(a), effective_unitary(b)), (name, i)
            else:
                assert tuple(a.params) == tuple(b.params), (name, i)
        # fused ops act on ascending qubit unions (ref dag.py:144-151)
        assert all(list(op.targets) == sorted(op.targets) for op in got.gates
                   if op.kind is GateKind.CUSTOM), name


def test_fusion_counts_at_baseline_configs():
    with open(os.path.join(GOLDEN, "fusion_stats.json")) as fh:
        stats = json.load(fh)
    for n in (20, 28, 30, 33, 36):
        c = gen.layered_circuit(n)
        f, rep = fuse(c, 2)
        assert [rep.original_gate_count, rep.fused_gate_count, rep.original_depth,
                rep.fused_depth] == stats[f"layered-{n}"], n
        assert depth(f) == rep.fused_depth
    f, rep = fuse(gen.qft_circuit(30), 2)
    assert [rep.original_gate_count, rep.fused_gate_count, rep.original_depth,
            rep.fused_depth] == stats["qft-30"]
    diag = sum(1 for g in f.gates
               if np.count_nonzero(effective_unitary(g) - np.diag(np.diag(effective_unitary(g)))) == 0)
    assert diag == stats["qft-30-diagonal"]
