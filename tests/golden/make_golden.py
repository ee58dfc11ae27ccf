"""Generate the golden fixtures from the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``aqsim`` from /root/reference/pkg/src and the reference tests'
own random-circuit fixture (``pkg/tests/conftest.py:19-85``), runs circuits on
``aqsim``'s ReferenceEngine (``engines.py:190-203``) and its fusion pass
(``dag.py:177-217``), and stores inputs + outputs as .npz next to this file.
The GPU box never runs this script; the tests only read its outputs.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
sys.path.insert(0, os.path.dirname(HERE))          # tests/ (golden_io)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))  # repo root

import aqsim  # noqa: E402
from aqsim import circuit as rc  # noqa: E402
from aqsim import dag as rdag  # noqa: E402
from aqsim.engines import get_engine  # noqa: E402
import conftest as refconf  # noqa: E402  (reference tests' fixtures)

from golden_io import encode  # noqa: E402
from paper_2604_03816_b200 import generators as mygen  # noqa: E402

REF = get_engine("reference")


def to_ref(c):
    return rc.Circuit(c.num_qubits, [rc.GateOp(rc.GateKind(g.kind.value), g.targets,
                                                g.params, g.matrix) for g in c.gates], c.name)


def run_both(c):
    return (REF.run_circuit(c, rc.Precision.DOUBLE).amplitudes.copy(),
            REF.run_circuit(c, rc.Precision.SINGLE).amplitudes.copy())


def main():
    # 1. random circuits drawn by the reference tests' own generator (seed 1234,
    #    the `rng` fixture of conftest.py:105-107), all 16 gate kinds incl. CUSTOM
    out = {}
    rng = np.random.default_rng(1234)
    count = 0
    for i in range(48):
        n = int(rng.integers(1, 9))
        g = int(rng.integers(1, 61))
        c = refconf.random_circuit(rng, n, g)
        s128, s64 = run_both(c)
        encode(f"c{i}_", c, out)
        out[f"c{i}_c128"] = s128
        out[f"c{i}_c64"] = s64
        if n <= 6:
            out[f"c{i}_kron"] = refconf.oracle_state(c)
        count += 1
    out["count"] = np.int64(count)
    np.savez_compressed(os.path.join(HERE, "random_circuits.npz"), **out)

    # 2. fused circuits: fusion output + reference states of fused and unfused
    out = {}
    cases = {
        "layered10_w2": (mygen.layered_circuit(10), 2),
        "layered9_w3": (mygen.layered_circuit(9, layers=6, seed=3), 3),
        "qft10_w2": (to_ref(mygen.qft_circuit(10)), 2),
        "qft9_w3": (to_ref(mygen.qft_circuit(9)), 3),
        "su2_8_w2": (aqsim.random_su2_circuit(8, 80, seed=8), 2),
        "ghz8_w2": (aqsim.ghz_circuit(8), 2),
    }
    names = []
    for name, (c, w) in cases.items():
        c = to_ref(c) if not isinstance(c, rc.Circuit) else c
        fused, rep = rdag.fuse(c, w)
        s128, s64 = run_both(fused)
        u128, _ = run_both(c)
        encode(f"{name}_orig_", c, out)
        encode(f"{name}_fused_", fused, out)
        out[f"{name}_c128"] = s128
        out[f"{name}_c64"] = s64
        out[f"{name}_unfused_c128"] = u128
        out[f"{name}_width"] = np.int64(w)
        names.append(name)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "fused_circuits.npz"), **out)

    # 3. fusion structure at the BASELINE configs (counts/depths only)
    stats = {}
    for n in (20, 28, 30, 33, 36):
        c = to_ref(mygen.layered_circuit(n))
        f, r = rdag.fuse(c, 2)
        stats[f"layered-{n}"] = [r.original_gate_count, r.fused_gate_count,
                                 r.original_depth, r.fused_depth]
    f, r = rdag.fuse(aqsim.qft_circuit(30), 2)
    stats["qft-30"] = [r.original_gate_count, r.fused_gate_count, r.original_depth,
                       r.fused_depth]
    stats["qft-30-diagonal"] = int(sum(
        1 for g in f.gates
        if np.count_nonzero(np.abs(rc.effective_unitary(g) - np.diag(np.diag(
            rc.effective_unitary(g)))) ) == 0))
    with open(os.path.join(HERE, "fusion_stats.json"), "w") as fh:
        json.dump(stats, fh, indent=1, sort_keys=True)
    print(json.dumps(stats))


if __name__ == "__main__":
    main()
