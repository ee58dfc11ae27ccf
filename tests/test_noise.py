"""Density-matrix noise arm (ref pkg/src/aqsim/noise.py:61-102).

CPU: the oracle restatement against the reference's own outputs
(tests/golden/noise_golden.npz), and the vec(rho) superoperator circuit run
by the state-vector oracle against it (the lowering, without a GPU).
GPU: ``paper_2604_03816_b200.noise.evolve_noisy`` (one planned 2n-qubit
circuit on the device) against the golden density matrices, c128 tolerance.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from golden_io import decode
from oracle import noise_oracle as nor
from oracle import sv_oracle as orc
from paper_2604_03816_b200 import noise

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "noise_golden.npz")


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


def cases(z):
    for name in z["names"]:
        c = decode(f"{name}_", z)
        for i, p in enumerate(z["ps"]):
            yield str(name), c, float(p), z[f"{name}_rho{i}"]


def test_oracle_matches_reference_fixtures(golden):
    for name, c, p, want in cases(golden):
        got = nor.evolve_noisy(c, p)
        assert np.abs(got - want).max() <= 1e-13, (name, p)


def test_superoperator_circuit_on_the_state_vector_oracle(golden):
    """vec(rho) as a 2n-qubit state: U on rows, conj(U) on columns, the
    channel as a 4x4 superoperator on (q, q + n)."""
    for name, c, p, want in cases(golden):
        vc = noise.superoperator_circuit(c, p)
        dim = 1 << c.num_qubits
        vec = orc.run_circuit(vc, "double")
        rho = vec.reshape(dim, dim).T
        assert np.abs(rho - want).max() <= 1e-12, (name, p)


def test_errors_mirror_the_reference():
    from paper_2604_03816_b200 import generators as gen
    with pytest.raises(ValueError):
        noise.evolve_noisy(gen.ghz_circuit(9), 0.0)          # over the default cap 8
    with pytest.raises(ValueError):
        noise.evolve_noisy(gen.ghz_circuit(3), 1.5)
    with pytest.raises(ValueError):
        noise.evolve_noisy(gen.ghz_circuit(11), 0.0, qubit_cap=12)  # hard cap 10


@pytest.mark.gpu
def test_device_evolution_matches_reference(golden):
    from paper_2604_03816_b200 import B200Engine
    eng = B200Engine("noise-test")
    for name, c, p, want in cases(golden):
        rho = noise.evolve_noisy(c, p, engine=eng)
        assert np.abs(rho.matrix - want).max() <= 1e-12, (name, p)
        rho.validate()
    from paper_2604_03816_b200 import generators as gen
    c8 = gen.random_su2_circuit(8, 40, seed=3)
    rho = noise.evolve_noisy(c8, 0.02, engine=eng)
    assert np.abs(rho.matrix - nor.evolve_noisy(c8, 0.02)).max() <= 1e-12
    # 10 qubits (the reference's hard cap): a 20-qubit vec(rho) on the device;
    # p = 0: the diagonal is the state-vector probability vector (ref criterion 9)
    c = gen.random_su2_circuit(10, 40, seed=3)
    noise.evolve_noisy(c, 0.02, qubit_cap=10, engine=eng).validate()
    rho0 = noise.evolve_noisy(c, 0.0, qubit_cap=10, engine=eng)
    probs = np.abs(orc.run_circuit(c, "double")) ** 2
    assert np.abs(rho0.diagonal_probabilities() - probs).max() <= 1e-12


@pytest.mark.gpu
def test_noise_compare_cli(capsys):
    """`python -m paper_2604_03816_b200 noise-compare` (ref cli.py:384-417): at
    p = 0 the outcome distribution is the ideal one; fidelity falls with p."""
    import json
    from paper_2604_03816_b200.__main__ import main
    assert main(["noise-compare", "--widths", "2,3", "--p-values", "0.0,0.01,0.05"]) == 0
    rows = json.loads(capsys.readouterr().out)
    assert len(rows) == 6
    for r in rows:
        if r["p"] == 0.0:
            assert abs(r["f_cl_exact"] - 1.0) <= 1e-6 and r["tvd_exact"] <= 1e-6
    for w in (2, 3):
        f = [r["f_cl_exact"] for r in rows if r["width"] == w]
        assert f[0] >= f[1] >= f[2]
