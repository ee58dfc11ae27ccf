"""Golden fixtures for the density-matrix noise arm, produced by the REFERENCE
(``aqsim.noise.evolve_noisy``, ref pkg/src/aqsim/noise.py:61-102) on the
circuits of its acceptance criterion 9 (ref pkg/tests/test_acceptance.py:236-260).

    python tests/golden/make_noise_golden.py      (build container only)
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import aqsim  # noqa: E402
from aqsim import generators as rg  # noqa: E402
from aqsim.noise import evolve_noisy  # noqa: E402

from golden_io import encode  # noqa: E402

CIRCUITS = {
    "bell": rg.bell_circuit(),
    "ghz3": rg.ghz_circuit(3),
    "ghz5": rg.ghz_circuit(5),
    "qft4": rg.qft_circuit(4),
    "su2_5": rg.random_su2_circuit(5, 30, seed=21),
    "ansatz4": rg.ansatz_circuit(4, 2, seed=8),
}
PS = (0.0, 0.01, 0.05)


def main():
    out = {"names": np.array(list(CIRCUITS), dtype="U16"), "ps": np.array(PS)}
    for name, c in CIRCUITS.items():
        encode(f"{name}_", c, out)
        for i, p in enumerate(PS):
            out[f"{name}_rho{i}"] = evolve_noisy(c, p, check_steps=True).matrix
    np.savez_compressed(os.path.join(HERE, "noise_golden.npz"), **out)
    print("wrote noise_golden.npz", aqsim.__version__ if hasattr(aqsim, "__version__") else "")


if __name__ == "__main__":
    main()
