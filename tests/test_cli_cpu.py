"""CLI argument handling on CPU (no device work)."""
from paper_2604_03816_b200.__main__ import _load, main


def test_generator_specs():
    assert _load("qft-5", 0).num_qubits == 5
    assert len(_load("layered-6", 0).gates) == 14 * (6 + 3 + 6) - 7
    assert len(_load("random-4-9", 1).gates) == 9


def test_bad_spec_is_an_error(capsys):
    assert main(["run", "nonsense-spec"]) == 2
    assert "error" in capsys.readouterr().err
