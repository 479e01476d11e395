"""CPU tests of the noisy-trajectory host logic: Pauli-frame propagation
(trajectory_program) against a gate-by-gate numpy replay of the reference's
trajectory (noise.py:109-131, same Philox draws), and the fit arithmetic."""
import numpy as np
import pytest

import paper_2604_26423_b200 as L
from paper_2604_26423_b200.noise import _PAULI_BRANCH, trajectory_program
from paper_2604_26423_b200.rng import derive_rng


def _rx(a, q, theta):
    v = a.reshape(-1, 2, 1 << q)
    c, s = np.cos(theta / 2), -1j * np.sin(theta / 2)
    a0, a1 = v[:, 0, :].copy(), v[:, 1, :].copy()
    v[:, 0, :] = c * a0 + s * a1
    v[:, 1, :] = s * a0 + c * a1


def _rzz(a, i, j, theta):
    n = int(np.log2(a.size))
    z = np.arange(a.size)
    par = ((z >> i) ^ (z >> j)) & 1
    a *= np.where(par == 0, np.exp(-0.5j * theta), np.exp(0.5j * theta))


def _h(a, q):
    v = a.reshape(-1, 2, 1 << q)
    a0, a1 = v[:, 0, :].copy(), v[:, 1, :].copy()
    v[:, 0, :] = (a0 + a1) / np.sqrt(2)
    v[:, 1, :] = (a0 - a1) / np.sqrt(2)


def _pauli(a, code, q):
    v = a.reshape(-1, 2, 1 << q)
    a0, a1 = v[:, 0, :].copy(), v[:, 1, :].copy()
    if code == 1:
        v[:, 0, :], v[:, 1, :] = a1, a0
    elif code == 2:
        v[:, 0, :], v[:, 1, :] = -1j * a1, 1j * a0
    elif code == 3:
        v[:, 1, :] = -a1


def _gate_by_gate(circ, cfg, t):
    n = circ.num_qubits
    a = np.zeros(1 << n, dtype=np.complex128)
    a[0] = 1.0
    n_rzz = sum(g.kind == "RZZ" for g in circ.gates)
    rng = derive_rng(cfg.rng_seed, "trajectory", t)
    fire = rng.random(n_rzz) < _PAULI_BRANCH * cfg.epsilon
    codes = rng.integers(1, 16, size=n_rzz)
    k = 0
    for g in circ.gates:
        if g.kind == "H":
            _h(a, g.qubits[0])
        elif g.kind == "RX":
            _rx(a, g.qubits[0], g.theta)
        else:
            _rzz(a, g.qubits[0], g.qubits[1], g.theta)
            if fire[k]:
                pa, pb = divmod(int(codes[k]), 4)
                if pa:
                    _pauli(a, pa, g.qubits[0])
                if pb:
                    _pauli(a, pb, g.qubits[1])
            k += 1
    return np.abs(a) ** 2


def _propagated(n, phase, mixer, mask):
    a = np.full(1 << n, 2.0 ** (-n / 2), dtype=np.complex128)
    iu = [(i, j) for i in range(n) for j in range(i + 1, n)]
    for k in range(mixer.shape[0]):
        for e, (i, j) in enumerate(iu):
            _rzz(a, i, j, 2 * phase[k, e])
        for q in range(n):
            _rx(a, q, 2 * mixer[k, q])
    pr = np.abs(a) ** 2
    out = np.empty_like(pr)
    out[np.arange(pr.size) ^ mask] = pr
    return out


@pytest.mark.parametrize("n,p,eps,seed", [(4, 2, 0.3, 1), (5, 3, 0.2, 7), (6, 2, 0.5, 3)])
def test_pauli_frame_propagation_matches_gate_by_gate(n, p, eps, seed):
    circ = L.build_circuit(L.generate_instance(n, seed), L.LrQaoaParams(p=p))
    cfg = L.DepolarizingConfig(eps, trajectories=6, rng_seed=seed)
    fired = 0
    for t in range(cfg.trajectories):
        phase, mixer, mask = trajectory_program(circ, cfg, t)
        want = _gate_by_gate(circ, cfg, t)
        got = _propagated(n, phase, mixer, mask)
        np.testing.assert_allclose(got, want, atol=1e-13)
        fired += int(mask != 0) + int(np.any(mixer < 0) != np.any(mixer[0] < 0))
    assert fired > 0  # the cases do exercise X masks / flipped mixers


def test_zero_noise_program_is_the_ideal_circuit():
    circ = L.build_circuit(L.generate_instance(6, 2), L.LrQaoaParams(p=3))
    phase, mixer, mask = trajectory_program(circ, L.DepolarizingConfig(0.0), 0)
    lay = L.lower_circuit(circ)
    np.testing.assert_array_equal(phase, lay.phase)
    assert mask == 0 and np.all(mixer == lay.mixer[:, None])


def test_config_fit_and_overlap_arithmetic():
    with pytest.raises(L.ValidationError):
        L.DepolarizingConfig(1.5)
    with pytest.raises(L.ValidationError):
        L.DepolarizingConfig(0.1, trajectories=0)
    assert L.epsilon_accumulated(198, 0.01) == pytest.approx(1.98)
    fit = L.fit_k0([(x, 2.0 ** (-0.4 * x)) for x in (0.1, 0.5, 1.0, 2.0)] + [(3.0, -0.1)])
    assert fit.k0 == pytest.approx(0.4) and fit.r_squared == pytest.approx(1.0) and fit.n_excluded == 1
    with pytest.raises(L.FitError):
        L.fit_k0([(1.0, -0.2)])
    assert L.r_overlap(0.8, 0.6, 1.0) == pytest.approx(0.5)
    assert L.predict_r_overlap(0.5, 10, 0.1) == pytest.approx(2.0 ** -0.5)


def test_batched_programs_equal_per_trajectory_programs():
    from paper_2604_26423_b200.noise import batch_programs
    circ = L.build_circuit(L.generate_instance(7, 3), L.LrQaoaParams(p=4))
    cfg = L.DepolarizingConfig(0.15, trajectories=9, rng_seed=21)
    ph, mx, mk = batch_programs(circ, cfg)
    for t in range(cfg.trajectories):
        p1, m1, k1 = trajectory_program(circ, cfg, t)
        np.testing.assert_array_equal(ph[t], p1)
        np.testing.assert_array_equal(mx[t], m1)
        assert int(mk[t]) == k1
