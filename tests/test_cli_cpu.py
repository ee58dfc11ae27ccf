"""CLI argument handling on CPU (no device work)."""
from paper_2604_03816_b200.__main__ import _load, main


def test_generator_specs():
    assert _load("qft-5", 0).num_qubits == 5
    assert len(_load("layered-6", 0).gates) == 14 * (6 + 3 + 6) - 7
    assert len(_load("random-4-9", 1).gates) == 9


def test_bad_spec_is_an_error(capsys):
    assert main(["run", "nonsense-spec"]) == 2
    assert "error" in capsys.readouterr().err


def test_bench_fusion_no_exec(capsys):
    """bench-fusion (ref cli.py:340-381) reports the fusion depth reduction;
    --no-exec needs no device."""
    import json
    assert main(["bench-fusion", "--circuits", "qft-8,layered-10", "--no-exec"]) == 0
    rows = json.loads(capsys.readouterr().out)
    assert [r["circuit"] for r in rows] == ["qft-8", "layered-10"]
    assert all(r["fused_depth"] <= r["original_depth"] for r in rows)
