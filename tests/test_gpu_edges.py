"""GPU edge cases of the hot path: sizes around the tile boundary (the
whole-state kernel below one tile, exactly one tile, two tiles), the
smallest circuits, one shot, empty index arrays and the reference's input
errors (ValidationError) at the API boundary.  Against the oracle
(oracle/lrq_oracle.py) with the north_star tolerances."""
import numpy as np
import pytest

import paper_2604_26423_b200 as L
from oracle import lrq_oracle as O
from paper_2604_26423_b200 import _native

pytestmark = pytest.mark.gpu

TOL = {"fp64": 1e-10, "fp32": 1e-5}


@pytest.fixture(scope="module", autouse=True)
def _engine():
    from paper_2604_26423_b200.build import build
    build()
    assert _native.device_count() >= 1, "GPU tests need a CUDA device"


def _normwise(got, want):
    return float(np.linalg.norm(got.astype(np.complex128) - want) / np.linalg.norm(want))


# complex64 tiles hold 2^13 amplitudes, complex128 tiles 2^12: n = KA - 1
# (whole-state kernel), KA (one tile), KA + 1 and KA + 2 (two / four tiles)
@pytest.mark.parametrize("n,prec", [(2, "fp64"), (3, "fp32"), (11, "fp64"), (12, "fp64"), (13, "fp64"),
                                    (14, "fp64"), (12, "fp32"), (13, "fp32"), (14, "fp32"), (15, "fp32")])
@pytest.mark.parametrize("p", [1, 2])
def test_tile_boundary_sizes_match_the_oracle(n, prec, p):
    inst = L.solve_instance(L.generate_instance(n, 60 + n))
    sv = L.run_circuit(L.build_circuit(inst, L.LrQaoaParams(p=p)), prec)
    try:
        want = O.simulate(n, inst.weights(), p, "fp64")
        assert _normwise(sv.amps, want) < TOL[prec]
        r_want = O.expected_cut(n, inst.weights(), O.probabilities(want)) / inst.optimal_cut.value
        assert L.exact_expected_r(sv, inst) == pytest.approx(r_want, rel=TOL[prec])
        # one shot, and the same shot again for the same seed
        a, b = L.sample(sv, 1, rng_seed=5), L.sample(sv, 1, rng_seed=5)
        assert a.indices.shape == (1,) and a.indices.dtype == np.uint64 and a.indices[0] < (1 << n)
        assert np.array_equal(a.indices, b.indices)
    finally:
        sv.release()


def test_empty_and_degenerate_inputs():
    inst = L.generate_instance(10, 1)
    assert L.cut_values(inst, np.array([], dtype=np.uint64)).shape == (0,)
    sv = L.run_circuit(L.build_circuit(L.solve_instance(inst), L.LrQaoaParams(p=1)), "fp64")
    try:
        with pytest.raises(L.ValidationError):
            L.sample(sv, 0, rng_seed=1)
        with pytest.raises(L.ValidationError):
            L.exact_expected_r(sv, L.solve_instance(L.generate_instance(11, 1)))  # size mismatch
    finally:
        sv.release()
    with pytest.raises(L.StateError):  # r needs C*: an unsolved instance
        sv2 = L.run_circuit(L.build_circuit(inst, L.LrQaoaParams(p=1)), "fp64")
        try:
            L.exact_expected_r(sv2, inst)
        finally:
            sv2.release()
    with pytest.raises(L.ValidationError):
        L.generate_instance(1, 0)


def test_many_shots_follow_the_exact_distribution():
    """10^6 shots at n=16: every outcome's count against its exact
    probability (a G-test over the outcomes expected >= 20 times)."""
    n = 16
    inst = L.solve_instance(L.generate_instance(n, 7))
    sv = L.run_circuit(L.build_circuit(inst, L.LrQaoaParams(p=3)), "fp64")
    try:
        shots = L.sample(sv, 1_000_000, rng_seed=11).indices
        p = np.abs(O.simulate(n, inst.weights(), 3, "fp64")) ** 2
    finally:
        sv.release()
    counts = np.bincount(shots.astype(np.int64), minlength=1 << n).astype(float)
    exp = p / p.sum() * shots.size
    keep = exp >= 20
    obs_k, exp_k = counts[keep], exp[keep]
    obs_r, exp_r = counts[~keep].sum(), exp[~keep].sum()
    g = 2 * float(np.sum(np.where(obs_k > 0, obs_k * np.log(obs_k / exp_k), 0.0)))
    if exp_r > 0 and obs_r > 0:
        g += 2 * obs_r * np.log(obs_r / exp_r)
    df = int(keep.sum()) - (0 if exp_r > 0 else 1)
    from scipy import stats
    assert stats.chi2.sf(g, df) > 1e-3, (g, df)
