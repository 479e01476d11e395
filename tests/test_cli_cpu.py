"""CPU tests of the gen/simulate command line (host-side parts only)."""
import json
import os

import pytest

from paper_2604_26423_b200.cli import main

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_gen_without_solve_matches_reference_instance(tmp_path):
    out = tmp_path / "i.json"
    assert main(["gen", "--n", "12", "--seed", "7", "--out", str(out), "--solve-limit", "0"]) == 0
    got = json.loads(out.read_text())
    want = json.load(open(os.path.join(GOLDEN, "cli_n12_inst.json")))
    assert got["n"] == want["n"] and got["edges"] == want["edges"]  # same Philox weights, bit for bit
    assert got["optimal"] is None
    man = json.loads((tmp_path / "i.json.manifest.json").read_text())
    assert man["command"] == "gen" and str(out) in man["outputs"]


def test_simulate_input_errors_exit_2(tmp_path, capsys):
    assert main(["simulate", "--instance", str(tmp_path / "missing.json"), "--out", str(tmp_path / "r.json")]) == 2
    inst = os.path.join(GOLDEN, "cli_n12_inst.json")
    assert main(["simulate", "--instance", inst, "--out", str(tmp_path / "r.json"), "--mode", "noisy",
                 "--epsilon", "1.5"]) == 2
    assert "epsilon must lie in [0, 1]" in capsys.readouterr().err
    with pytest.raises(SystemExit):
        main(["simulate", "--instance", inst, "--out", str(tmp_path / "r.json"), "--precision", "fp16"])


def test_circuit_text_and_cost_model_match_reference():
    import paper_2604_26423_b200 as L
    circ = L.build_circuit(L.generate_instance(5, 1), L.LrQaoaParams(p=2))
    assert L.circuit_to_text(circ) == open(os.path.join(GOLDEN, "circuit_n5.txt")).read()
    assert L.hqc_cost(160, 2340, 40, 10) == pytest.approx(52.52)
    with pytest.raises(L.ValidationError):
        L.hqc_cost(1, 1, 1, 0)
