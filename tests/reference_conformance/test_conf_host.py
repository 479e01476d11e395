"""Host-only conformance: the reference's problem / circuit / rng / shard-plan
/ memory-budget tests that need no device (instance construction and
validation, schedules, gate lists, shard plans and exchange accounting,
frozen rng streams, the CapacityError contract)."""
import json

import numpy as np
import pytest

from paper_2604_26423_b200 import rng as lrng
from paper_2604_26423_b200.engine import check_memory, state_bytes
from paper_2604_26423_b200.problem import as_index, bitstring_to_index, complete_edge_list, index_to_bitstring


# --- test_problem.py ---------------------------------------------------------

def test_edge_list_and_instances(lq):
    """test_complete_edge_list_lexicographic, test_generate_instance_deterministic,
    test_generate_instance_weights_in_unit_interval, test_edges_normalized_to_sorted_order"""
    assert complete_edge_list(4) == [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]
    assert complete_edge_list(2) == [(0, 1)]
    a, b, c = lq.generate_instance(6, 42), lq.generate_instance(6, 42), lq.generate_instance(6, 43)
    assert a.edges == b.edges and a.seed == 42 and c.edges != a.edges
    ws = [w for _, _, w in lq.generate_instance(12, 7).edges]
    assert len(ws) == 66 and all(0.0 <= w <= 1.0 for w in ws)
    inst = lq.WmcInstance(3, ((2, 1, 0.25), (0, 1, 0.5), (2, 0, 1.0)))
    assert inst.edges == [(0, 1, 0.5), (0, 2, 1.0), (1, 2, 0.25)]


@pytest.mark.parametrize("n,edges", [
    (1, ()),
    (3, ((0, 1, 0.5), (0, 2, 1.0))),
    (3, ((0, 1, 0.5), (0, 2, 1.0), (1, 2, 0.25), (1, 2, 0.25))),
    (3, ((0, 1, 0.5), (0, 2, 1.0), (1, 2, 1.25))),
    (3, ((0, 1, 0.5), (0, 2, 1.0), (2, 2, 0.25))),
])
def test_bad_instances_rejected(lq, n, edges):
    """test_bad_instances_rejected"""
    with pytest.raises(lq.ValidationError):
        lq.WmcInstance(n, edges)


def test_bitstrings_and_index_forms(lq):
    """test_bitstring_encoding_vertex_zero_leftmost, test_as_index_accepts_all_forms"""
    assert [bitstring_to_index(s) for s in ("100", "010", "001")] == [1, 2, 4]
    assert index_to_bitstring(1, 3) == "100" and index_to_bitstring(6, 3) == "011"
    assert all(bitstring_to_index(index_to_bitstring(z, 5)) == z for z in range(32))
    for form in ("110", 3, [1, 1, 0], np.uint64(3)):
        assert as_index(form, 3) == 3
    for bad in ("11", 8):
        with pytest.raises(lq.ValidationError):
            as_index(bad, 3)


def test_weight_matrix_and_total(triangle):
    """test_weight_matrix_symmetric_zero_diagonal"""
    m = triangle.weight_matrix()
    np.testing.assert_array_equal(m, m.T)
    assert np.all(np.diag(m) == 0.0) and m[0, 2] == 1.0
    assert abs(triangle.total_weight() - 1.75) < 1e-15


def test_instance_json_roundtrip(lq, tmp_path):
    """test_save_load_roundtrip, test_load_unsolved_instance (solving is a
    device call; an optimal cut is attached by hand here)"""
    inst = lq.generate_instance(5, 13)
    solved = lq.WmcInstance(inst.num_vertices, inst.edges, inst.seed, lq.OptimalCut("10101", 1.0))
    path = tmp_path / "inst.json"
    lq.save_instance(solved, path)
    back = lq.load_instance(path)
    assert back == solved and back.optimal_cut == solved.optimal_cut
    assert set(json.loads(path.read_text())) == {"n", "seed", "edges", "optimal"}
    lq.save_instance(inst, path)
    assert lq.load_instance(path).optimal_cut is None


# --- test_circuit.py ---------------------------------------------------------

def test_schedule_values(lq):
    """test_schedule_p3_default_ramps, test_schedule_endpoints"""
    s = lq.build_schedule(lq.LrQaoaParams(p=3))
    np.testing.assert_allclose(s.betas, (0.2, 2.0 / 15.0, 1.0 / 15.0))
    np.testing.assert_allclose(s.gammas, (1.0 / 15.0, 2.0 / 15.0, 0.2))
    assert s.p == 3
    for p in (1, 2, 7, 50):
        s = lq.build_schedule(lq.LrQaoaParams(p=p, delta_beta=0.3, delta_gamma=0.15))
        assert s.betas[0] == pytest.approx(0.3) and s.gammas[-1] == pytest.approx(0.15)
        assert s.betas[-1] == pytest.approx(0.3 / p) and s.gammas[0] == pytest.approx(0.15 / p)
        assert all(a > b for a, b in zip(s.betas, s.betas[1:]))
        assert all(a < b for a, b in zip(s.gammas, s.gammas[1:]))


@pytest.mark.parametrize("kw", [{"p": 0}, {"p": -1}, {"p": 2.0}, {"p": 3, "delta_beta": 0.0},
                                {"p": 3, "delta_gamma": -0.2}, {"p": 3, "delta_beta": float("nan")}])
def test_bad_params_rejected(lq, kw):
    """test_bad_params_rejected"""
    with pytest.raises(lq.ValidationError):
        lq.LrQaoaParams(**kw)


def test_gate_sequence_and_counts(lq, triangle):
    """test_build_circuit_gate_sequence, test_built_gate_totals_match_formula,
    test_gate_counts_published_sizes, test_gate_counts_validation"""
    circ = lq.build_circuit(triangle, lq.LrQaoaParams(p=2))
    assert circ.num_qubits == 3 and circ.p == 2
    assert [g.kind for g in circ.gates] == ["H"] * 3 + (["RZZ"] * 3 + ["RX"] * 3) * 2
    for layer in range(2):
        base = 3 + 6 * layer
        for k, (i, j, w) in enumerate(triangle.edges):
            g = circ.gates[base + k]
            assert g.qubits == (i, j) and g.theta == pytest.approx(2.0 * circ.schedule.gammas[layer] * w)
        for k in range(3):
            g = circ.gates[base + 3 + k]
            assert g.kind == "RX" and g.qubits == (k,)
            assert g.theta == pytest.approx(-2.0 * circ.schedule.betas[layer])
    c5 = lq.build_circuit(lq.generate_instance(5, 0), lq.LrQaoaParams(p=4))
    n1, n2 = lq.gate_counts(5, 4)
    assert sum(g.kind in ("H", "RX") for g in c5.gates) == n1 and sum(g.kind == "RZZ" for g in c5.gates) == n2
    assert lq.gate_counts(48, 3) == (192, 3384) and lq.gate_counts(93, 3) == (372, 12834)
    assert lq.gate_counts(40, 3) == (160, 2340)
    for bad in ((1, 3), (5, 0)):
        with pytest.raises(lq.ValidationError):
            lq.gate_counts(*bad)


@pytest.mark.parametrize("kind,qubits,theta", [("CZ", (0, 1), 0.1), ("H", (0, 1), None), ("RX", (0,), None),
                                               ("H", (0,), 0.1), ("RZZ", (1, 1), 0.1), ("RZZ", (0,), 0.1)])
def test_bad_gates_rejected(lq, kind, qubits, theta):
    """test_bad_gates_rejected, test_circuit_rejects_out_of_range_qubit"""
    with pytest.raises(lq.ValidationError):
        lq.GateOp(kind, qubits, theta)
    with pytest.raises(lq.ValidationError):
        lq.CircuitIR(num_qubits=2, gates=[lq.GateOp("H", (2,))])


def test_hqc_and_text(lq, triangle):
    """test_hqc_cost_formula, test_hqc_cost_validation, test_circuit_to_text_stable"""
    assert lq.hqc_cost(160, 2340, 40, 10) == pytest.approx(52.52, abs=1e-12)
    assert lq.hqc_cost(0, 0, 0, 1) == pytest.approx(5.0)
    for bad in ((-1, 0, 0, 1), (0, 0, 0, 0)):
        with pytest.raises(lq.ValidationError):
            lq.hqc_cost(*bad)
    circ = lq.build_circuit(triangle, lq.LrQaoaParams(p=1))
    text = lq.circuit_to_text(circ)
    lines = text.splitlines()
    assert text == lq.circuit_to_text(circ) and text.endswith("\n")
    assert lines[0] == "H 0" and lines[3].startswith("RZZ ") and lines[3].endswith(" 0 1")
    assert lines[6].startswith("RX ") and float(lines[3].split()[1]) == circ.gates[3].theta


# --- test_rng.py -------------------------------------------------------------

def test_rng_streams(lq):
    """test_stream_codes_are_frozen, test_same_stream_same_draws,
    test_streams_are_independent, test_seed_wraps_to_64_bits,
    test_unknown_stream_rejected, test_derive_seed_is_deterministic_uint64"""
    assert lrng._STREAMS == {"instance": 0, "shots": 1, "trajectory": 2, "uniform": 3, "resample": 4,
                             "classify": 5, "sweep": 6, "ideal": 7}
    np.testing.assert_array_equal(lrng.derive_rng(12, "shots", 4).random(8), lrng.derive_rng(12, "shots", 4).random(8))
    base = lrng.derive_rng(12, "shots", 0).random(4)
    for stream, idx in (("shots", 1), ("trajectory", 0), ("resample", 0)):
        assert not np.array_equal(base, lrng.derive_rng(12, stream, idx).random(4))
    np.testing.assert_array_equal(lrng.derive_rng(5, "instance").random(4),
                                  lrng.derive_rng(5 + (1 << 64), "instance").random(4))
    with pytest.raises(lq.ValidationError):
        lrng.derive_rng(0, "nope")
    s1 = lrng.derive_seed(3, "classify", 0)
    assert s1 == lrng.derive_seed(3, "classify", 0) and 0 <= s1 < (1 << 64)
    assert lrng.derive_seed(3, "classify", 1) != s1


# --- test_engine.py (host-only parts) -----------------------------------------

def test_precision_state_bytes_and_budget(lq, monkeypatch):
    """test_precision_coerce, test_state_bytes, test_capacity_error_names_requirement,
    test_memory_budget_env_override (check_memory part), test_explicit_budget_beats_env"""
    assert lq.Precision.coerce("fp32") is lq.Precision.FP32
    assert lq.Precision.coerce(lq.Precision.FP64) is lq.Precision.FP64
    with pytest.raises(lq.ValidationError):
        lq.Precision.coerce("fp16")
    assert state_bytes(33, lq.Precision.FP32) == 68719476736 and state_bytes(3, lq.Precision.FP64) == 128
    monkeypatch.delenv("LRQBENCH_MEMORY_BYTES", raising=False)
    with pytest.raises(lq.CapacityError, match=r"68719476736 bytes \(64\.0 GiB\)"):
        check_memory(33, lq.Precision.FP32)  # the reference's 4 GiB default budget
    monkeypatch.setenv("LRQBENCH_MEMORY_BYTES", str(1 << 20))
    with pytest.raises(lq.CapacityError):
        check_memory(18, lq.Precision.FP64)
    check_memory(16, lq.Precision.FP32)
    monkeypatch.setenv("LRQBENCH_MEMORY_BYTES", "1")
    check_memory(10, lq.Precision.FP32, budget=1 << 20)


def test_zero_state_over_env_budget_raises_before_the_device(lq, monkeypatch):
    """test_memory_budget_env_override: zero_state(18, fp64) over a 1 MiB budget"""
    monkeypatch.setenv("LRQBENCH_MEMORY_BYTES", str(1 << 20))
    with pytest.raises(lq.CapacityError):
        lq.zero_state(18, "fp64")


# --- test_sharded.py (plans and accounting) ------------------------------------

def test_shard_plans(lq):
    """test_plan_shards_published_sizes, test_plan_for_shard_count, test_plan_shards_validation"""
    assert lq.plan_shards(46, 33).num_shards == 8192 and lq.plan_shards(48, 34).num_shards == 16384
    p = lq.plan_shards(5, 3)
    assert (p.num_shards, p.shard_len) == (4, 8)
    p = lq.plan_for_shard_count(12, 8)
    assert (p.nq_local, p.num_shards) == (9, 8)
    for bad in ((12, 3), (3, 8)):
        with pytest.raises(lq.ValidationError):
            lq.plan_for_shard_count(*bad)
    for bad in ((5, 0), (5, 6)):
        with pytest.raises(lq.ValidationError):
            lq.plan_shards(*bad)


def test_exchange_steps_and_volume(lq):
    """test_local_gate_needs_no_exchange, test_global_gate_single_step,
    test_mixed_gate_slot_skips_local_operand, test_two_global_gate_two_steps,
    test_gate_too_large_for_shard, test_exchange_volume_hand_count,
    test_exchange_volume_counts_two_global_gates_twice"""
    plan = lq.plan_shards(6, 3)
    assert lq.exchange_steps(lq.GateOp("RX", (2,), 0.1), plan) == []
    assert lq.exchange_steps(lq.GateOp("RZZ", (0, 2), 0.1), plan) == []
    (st,) = lq.exchange_steps(lq.GateOp("RX", (4,), 0.1), plan)
    assert (st.global_qubit, st.pair_bit, st.local_slot, st.amps_per_shard) == (4, 1, 2, 4)
    assert st.partner(0b000) == 0b010
    assert sorted(st.pairs(plan.num_shards)) == [(0, 2), (1, 3), (4, 6), (5, 7)]
    assert lq.exchange_steps(lq.GateOp("RZZ", (2, 5), 0.1), plan)[0].local_slot == 1
    steps = lq.exchange_steps(lq.GateOp("RZZ", (3, 5), 0.1), plan)
    assert [s.global_qubit for s in steps] == [5, 3] and [s.local_slot for s in steps] == [2, 1]
    with pytest.raises(lq.ValidationError):
        lq.exchange_steps(lq.GateOp("RZZ", (2, 3), 0.1), lq.plan_shards(4, 1))
    one = lq.CircuitIR(num_qubits=4, gates=[lq.GateOp("RX", (3,), 0.5)])
    assert lq.exchange_volume(one, lq.plan_shards(4, 3)) == 8
    two = lq.CircuitIR(num_qubits=4, gates=[lq.GateOp("RZZ", (2, 3), 0.5)])
    assert lq.exchange_volume(two, lq.plan_shards(4, 2)) == 2 * lq.exchange_volume(one, lq.plan_shards(4, 2))


def test_sweep_config_validation(lq):
    """test_sweep_config_validation"""
    for kw in ({"mode": "weak"}, {"mode": "strong", "nq": None}, {"mode": "size", "nq_values": ()},
               {"mode": "strong", "nq": 8, "repeat": 0}):
        with pytest.raises(lq.ValidationError):
            lq.SweepConfig(**kw)


def test_acceptance_08_published_formulas(lq):
    """test_acceptance.py test_08_published_count_and_cost_formulas"""
    assert lq.gate_counts(48, 3) == (192, 3384) and lq.gate_counts(93, 3) == (372, 12834)
    assert lq.plan_shards(46, 33).num_shards == 8192 and lq.plan_shards(48, 34).num_shards == 16384
    assert abs(lq.hqc_cost(160, 2340, 40, 10) - 52.52) < 1e-9
