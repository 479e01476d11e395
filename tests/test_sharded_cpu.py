"""CPU tests of the sharded drop-in's host logic (mirrors the reference's
test_sharded.py: plan sizes and validation, the per-gate exchange
accounting, the timing CSV schema, sweep-config validation), plus the remap
volume of this engine's distributed plan and the in-process shard group's
creation contract (no device work)."""
import csv
import io

import numpy as np
import pytest

import paper_2604_26423_b200 as L
from paper_2604_26423_b200 import _native
from paper_2604_26423_b200.sharded import TIMING_CSV_FIELDS, _flips, _rows_from_timings


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_2604_26423_b200.build import build

    build()


def test_plan_sizes_and_validation():
    assert L.plan_shards(46, 33).num_shards == 8192
    plan = L.plan_shards(5, 3)
    assert (plan.num_shards, plan.shard_len) == (4, 8)
    plan = L.plan_for_shard_count(12, 8)
    assert (plan.nq_local, plan.num_shards) == (9, 8)
    for bad in [(12, 3), (3, 8)]:
        with pytest.raises(L.ValidationError):
            L.plan_for_shard_count(*bad)
    for bad in [(5, 0), (5, 6), (0, 1)]:
        with pytest.raises(L.ValidationError):
            L.plan_shards(*bad)


def test_reference_exchange_accounting():
    plan = L.plan_shards(6, 3)
    assert L.exchange_steps(L.GateOp("RX", (2,), 0.1), plan) == []
    (step,) = L.exchange_steps(L.GateOp("RX", (4,), 0.1), plan)
    assert (step.global_qubit, step.pair_bit, step.local_slot, step.amps_per_shard) == (4, 1, 2, 4)
    assert sorted(step.pairs(plan.num_shards)) == [(0, 2), (1, 3), (4, 6), (5, 7)]
    (step,) = L.exchange_steps(L.GateOp("RZZ", (2, 5), 0.1), plan)
    assert step.local_slot == 1
    steps = L.exchange_steps(L.GateOp("RZZ", (3, 5), 0.1), plan)
    assert [s.global_qubit for s in steps] == [5, 3] and [s.local_slot for s in steps] == [2, 1]
    with pytest.raises(L.ValidationError):
        L.exchange_steps(L.GateOp("RZZ", (2, 3), 0.1), L.plan_shards(4, 1))
    one = L.CircuitIR(num_qubits=4, gates=[L.GateOp("RX", (3,), 0.5)])
    two = L.CircuitIR(num_qubits=4, gates=[L.GateOp("RZZ", (2, 3), 0.5)])
    assert L.exchange_volume(one, L.plan_shards(4, 3)) == 8
    assert L.exchange_volume(two, L.plan_shards(4, 2)) == 2 * L.exchange_volume(one, L.plan_shards(4, 2))


@pytest.mark.parametrize("n,G,p,prec", [(16, 2, 3, "fp64"), (17, 4, 2, "fp64"), (20, 8, 4, "fp32")])
def test_remap_volume_vs_reference_volume(n, G, p, prec):
    inst = L.generate_instance(n, 1)
    circ = L.build_circuit(inst, L.LrQaoaParams(p=p))
    plan = L.plan_for_shard_count(n, G)
    remaps = p  # one per layer; an odd p ends in the swapped layout (no restoring remap)
    assert L.remap_volume(circ, plan, prec) == remaps * (G - 1) * (1 << n) // G
    # the per-layer remap moves far less than the reference's per-gate swaps
    assert L.remap_volume(circ, plan, prec) * 4 < L.exchange_volume(circ, plan)


def test_remap_volume_counts_the_flip_exchange():
    inst = L.generate_instance(16, 1)
    plan = L.plan_for_shard_count(16, 2)
    flip = L.build_circuit(inst, L.LrQaoaParams(p=2, delta_beta=1.2))  # beta_0 = 1.2 > pi/4
    lay = L.lower_circuit(flip)
    assert _flips(lay.mixer) == 1
    assert L.remap_volume(flip, plan, "fp64") == 2 * (1 << 16) // 2 + (1 << 16)
    # shards below one tile run dense: nothing moves
    small = L.build_circuit(L.generate_instance(8, 1), L.LrQaoaParams(p=2))
    assert L.remap_volume(small, L.plan_for_shard_count(8, 4)) == 0


def test_timing_rows_and_csv_schema():
    per_shard = [([1.0, 2.0, 0.5, 3.0], "PTFX"), ([1.5, 1.0, 0.25, 3.5], "PTFX")]
    rows = _rows_from_timings(per_shard, 16, 2)
    assert [r.kind for r in rows] == list("PTFX")
    assert rows[0].compute_s == pytest.approx(1.5e-3) and rows[0].exchange_s == 0.0
    assert rows[1].exchange_s == pytest.approx(2e-3) and rows[1].amps_exchanged == 1 << 15
    assert rows[3].amps_exchanged == 1 << 16
    rec = L.TimingRecord(nq=16, p=1, num_shards=2, wall_seconds=0.1, gates=rows)
    assert rec.amps_exchanged == (1 << 15) + (1 << 16)
    buf = io.StringIO()
    L.write_timing_csv([rec], buf)
    out = list(csv.reader(io.StringIO(buf.getvalue())))
    assert tuple(out[0]) == TIMING_CSV_FIELDS
    assert len(out) == 1 + len(rows)
    for row in out[1:]:
        assert row[0] == "16" and row[2] == "2"
        float(row[5]), float(row[6]), int(row[7])


def test_sweep_config_validation():
    with pytest.raises(L.ValidationError):
        L.SweepConfig(mode="weak")
    with pytest.raises(L.ValidationError):
        L.SweepConfig(mode="strong", nq=None)
    with pytest.raises(L.ValidationError):
        L.SweepConfig(mode="size", nq_values=())
    with pytest.raises(L.ValidationError):
        L.SweepConfig(mode="strong", nq=7, repeat=0)


def test_shard_group_contract():
    with pytest.raises(L.ValidationError):
        _native.ShardGroup(3)
    g = _native.ShardGroup(4)
    g.abort()  # breaking an empty group is allowed
    g.close()
    with pytest.raises(L.StateError):
        _ = g.handle


def test_run_circuit_sharded_validates_before_device_work():
    circ = L.build_circuit(L.generate_instance(5, 0), L.LrQaoaParams(p=1))
    with pytest.raises(L.ValidationError):
        L.run_circuit_sharded(circ, L.plan_shards(6, 3))
    circ = L.build_circuit(L.generate_instance(20, 0), L.LrQaoaParams(p=1))
    with pytest.raises(L.CapacityError):
        L.run_circuit_sharded(circ, L.plan_for_shard_count(20, 2), "fp64", memory_budget=1 << 20)
    assert np.isfinite(L.lower_circuit(circ).mixer).all()
