"""GPU parity at BASELINE.json's full single-GPU sizes, through properties
that do not need the (infeasible) CPU oracle at 2^32-2^33 amplitudes:

* configs[2] (n=32, p=10; the bench workload, 32 GiB in complex64) and the
  1-GPU point of configs[3] (n=33, p=3; 128 GiB in complex128): the
  complex64 run against the complex128 run of the same circuit;
* norm (sum of probabilities from the fused final pass) to 1e-12 in
  complex128 and 1e-5 in complex64;
* exact r agreeing to the complex64 tolerance (1e-5 relative);
* the max cut found by the fused final pass equals C* of the exhaustive GPU
  search, and is the same state in both precisions;
* the sampled r within 4 standard errors of the exact r.
"""
import math

import pytest

import paper_2604_26423_b200 as L
from paper_2604_26423_b200 import _native

pytestmark = pytest.mark.gpu

BUDGET = 1 << 40


@pytest.fixture(scope="module", autouse=True)
def _engine():
    from paper_2604_26423_b200.build import build
    build()
    assert _native.device_count() >= 1, "GPU tests need a CUDA device"


@pytest.mark.parametrize("n,p", [(32, 10), (33, 3)])
def test_full_size_complex64_against_complex128(n, p):
    inst = L.solve_instance(L.generate_instance(n, 1), limit=n)
    # built from the unsolved instance: the fused final pass runs its own
    # max-cut search, checked below against the exhaustive search's C*
    circ = L.build_circuit(L.generate_instance(n, 1), L.LrQaoaParams(p=p))
    out = {}
    for prec in ("fp32", "fp64"):
        sv = L.run_circuit(circ, prec, BUDGET)
        red = sv.device_state.reduce()
        shots = L.sample(sv, 4000, rng_seed=1) if prec == "fp32" else None
        out[prec] = (L.exact_expected_r(sv, inst), red, shots)
        sv.release()
        _native.drain_pool()
    (r32, red32, shots), (r64, red64, _) = out["fp32"], out["fp64"]
    assert abs(red64.sum_p - 1.0) < 1e-12
    assert abs(red32.sum_p - 1.0) < 1e-5
    assert r32 == pytest.approx(r64, rel=1e-5)
    assert red32.argmax_cut == red64.argmax_cut
    assert float(L.cut_values(inst, [red64.argmax_cut])[0]) == inst.optimal_cut.value
    ratios = L.shot_ratios(inst, shots)
    se = ratios.std() / math.sqrt(len(ratios))
    assert abs(ratios.mean() - r64) < 4 * se


def test_full_size_distributed_plan_matches_dense():
    """The distributed plan (rank-local phase fields, a fused remap per
    layer, the rank-partitioned reductions and sampler) at the bench size:
    n=32 on 8 in-process shards of 2^29 amplitudes against the dense run."""
    n, G, p = 32, 8, 4
    inst = L.solve_instance(L.generate_instance(n, 1), limit=n)
    circ = L.build_circuit(inst, L.LrQaoaParams(p=p))
    sv, rec = L.run_circuit_sharded(circ, L.plan_for_shard_count(n, G), "fp32", BUDGET)
    try:
        assert isinstance(sv, L.ShardedStateVector)
        assert "Y" in [g.kind for g in rec.gates]  # the remaps ran fused
        r_sh = L.exact_expected_r(sv, inst)
        shots_sh = L.sample(sv, 2000, rng_seed=2)
    finally:
        sv.release()
    dense = L.run_circuit(circ, "fp32", BUDGET)
    r_de = L.exact_expected_r(dense, inst)
    shots_de = L.sample(dense, 2000, rng_seed=2)
    dense.release()
    assert r_sh == pytest.approx(r_de, rel=1e-5)
    # at 2^32 outcomes complex64 rounding moves CDF boundaries across many
    # states, so shots need not coincide; both sample the same distribution
    for shots in (shots_sh, shots_de):
        ratios = L.shot_ratios(inst, shots)
        assert abs(ratios.mean() - r_de) < 4 * ratios.std() / math.sqrt(len(ratios))


def test_largest_one_gpu_complex64_state():
    """n=34 complex64 (128 GiB, 2^21 tiles): the largest complex64 state one
    B200 holds.  Norm, the fused max-cut search against the exhaustive one's
    C*, and sampled r within 4 SE of the exact r."""
    n, p = 34, 2
    inst = L.solve_instance(L.generate_instance(n, 1), limit=n)
    sv = L.run_circuit(L.build_circuit(L.generate_instance(n, 1), L.LrQaoaParams(p=p)), "fp32", BUDGET)
    try:
        red = sv.device_state.reduce()
        assert abs(red.sum_p - 1.0) < 1e-5
        assert float(L.cut_values(inst, [red.argmax_cut])[0]) == inst.optimal_cut.value
        r = L.exact_expected_r(sv, inst)
        ratios = L.shot_ratios(inst, L.sample(sv, 4000, rng_seed=2))
        assert abs(ratios.mean() - r) < 4 * ratios.std() / math.sqrt(len(ratios))
    finally:
        sv.release()
        _native.drain_pool()
