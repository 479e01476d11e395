"""GPU tests of the batched noisy trajectories against the reference's own
noise.py results (tests/golden/noise.npz, make_golden_noise.py) and its
zero-noise identities (test_noise.py:77-95)."""
import numpy as np
import pytest

import paper_2604_26423_b200 as L
from paper_2604_26423_b200 import _native

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _engine():
    from paper_2604_26423_b200.build import build
    build()
    assert _native.device_count() >= 1


@pytest.mark.parametrize("case", range(6))
def test_noisy_results_match_reference(golden, case):
    g = golden("noise.npz")
    n, p, T, seed = (int(x) for x in g[f"meta_{case}"])
    eps, prec = float(g[f"eps_{case}"]), str(g[f"prec_{case}"])
    inst = L.solve_instance(L.generate_instance(n, seed))
    circ = L.build_circuit(inst, L.LrQaoaParams(p=p))
    cfg = L.DepolarizingConfig(eps, trajectories=T, rng_seed=seed)
    probs = L.noisy_expected_probs(circ, cfg, prec)
    want = g[f"probs_{case}"]
    tol = 1e-12 if prec == "fp64" else 1e-5
    assert np.abs(probs - want).max() <= tol * want.max()
    r = L.noisy_expected_r(circ, inst, cfg, prec)
    assert r == pytest.approx(float(g[f"r_{case}"]), rel=tol)
    shots = L.run_noisy_ensemble(circ, cfg, 50, prec)
    assert shots.source == f"noisy(epsilon={eps:g}, trajectories={T})"
    if prec == "fp64":
        np.testing.assert_array_equal(shots.indices, g[f"shots_{case}"])
    else:
        assert np.mean(shots.indices == g[f"shots_{case}"]) > 0.97


def test_zero_noise_matches_noiseless_exactly():
    inst = L.generate_instance(6, 7)
    circ = L.build_circuit(inst, L.LrQaoaParams(p=3))
    sv = L.run_circuit(circ, "fp32")
    noisy = L.noisy_expected_probs(circ, L.DepolarizingConfig(0.0, trajectories=1), "fp32")
    np.testing.assert_array_equal(noisy, sv.probabilities())
    baseline = L.sample(sv, 200, rng_seed=5)
    ens = L.run_noisy_ensemble(circ, L.DepolarizingConfig(0.0, trajectories=1, rng_seed=5), 200, "fp32")
    np.testing.assert_array_equal(ens.indices, baseline.indices)


def test_noise_degrades_r_and_probs_normalised():
    inst = L.solve_instance(L.generate_instance(8, 4))
    circ = L.build_circuit(inst, L.LrQaoaParams(p=3))
    rs = [L.noisy_expected_r(circ, inst, L.DepolarizingConfig(e, trajectories=64, rng_seed=1), "fp64")
          for e in (0.0, 0.02, 0.2)]
    assert rs[0] > rs[1] > rs[2] > L.random_baseline_expectation(inst) - 0.05
    pr = L.noisy_expected_probs(circ, L.DepolarizingConfig(0.1, trajectories=32, rng_seed=2), "fp32")
    assert abs(pr.sum() - 1.0) < 1e-5


@pytest.mark.parametrize("n,p,eps,prec", [(14, 2, 0.05, "fp64"), (15, 3, 0.02, "fp32"), (16, 2, 0.2, "fp64"),
                                          (21, 3, 0.02, "fp64"), (24, 2, 0.01, "fp32")])
def test_above_tile_trajectories_match_gate_by_gate(n, p, eps, prec):
    """n above the tile: fused engine runs with per-qubit mixer signs + X
    string; checked per trajectory against the same trajectory replayed gate
    by gate on the GPU (lrq_apply_gate, the reference kernels' arithmetic)."""
    from paper_2604_26423_b200.noise import _PAULI_BRANCH
    from paper_2604_26423_b200.rng import derive_rng
    inst = L.generate_instance(n, 5)
    circ = L.build_circuit(inst, L.LrQaoaParams(p=p))
    T = 3
    cfg = L.DepolarizingConfig(eps, trajectories=T, rng_seed=8)
    probs = L.noisy_expected_probs(circ, cfg, prec)
    n_rzz = sum(g.kind == "RZZ" for g in circ.gates)
    acc = np.zeros(1 << n)
    for t in range(T):
        rng = derive_rng(cfg.rng_seed, "trajectory", t)
        fire = rng.random(n_rzz) < _PAULI_BRANCH * eps
        codes = rng.integers(1, 16, size=n_rzz)
        sv = L.zero_state(n, prec)
        k = 0
        for g in circ.gates:
            L.apply_gate(sv, g)
            if g.kind == "RZZ":
                if fire[k]:
                    # up to global phases: X = i RX(pi), Z = H X H, Y = X Z
                    for q, pc in zip(g.qubits, divmod(int(codes[k]), 4)):
                        if pc in (2, 3):
                            L.apply_h(sv, q)
                            L.apply_rx(sv, np.pi, q)
                            L.apply_h(sv, q)
                        if pc in (1, 2):
                            L.apply_rx(sv, np.pi, q)
                k += 1
        a = sv.amps.astype(np.complex128)
        acc += a.real ** 2 + a.imag ** 2
        sv.release()
    want = acc / T
    tol = 1e-12 if prec == "fp64" else 2e-6
    assert np.abs(probs - want).max() <= tol * want.max()
    shots = L.run_noisy_ensemble(circ, cfg, 40, prec)
    assert len(shots) == 3 * 40
