"""Two-qubit depolarizing noise via Monte Carlo Pauli trajectories (GPU).

Drop-in for lrqbench noise.py.  The reference runs
each trajectory gate by gate: after every RZZ, with probability 15 eps / 16,
one of the 15 non-identity two-qubit Paulis (noise.py:109-131).  Here the
Paulis are propagated to the end of the circuit on the host, which turns a
trajectory back into an LR-QAOA circuit the engine runs fused:

* an X or Y on qubit a anticommutes with Z_a: every later RZZ on an edge with
  exactly one flipped endpoint runs with the opposite angle;
* a Z or Y on qubit a anticommutes with X_a: every later RX(a) runs with the
  opposite angle;
* what is left at the end is a Pauli string whose X part permutes the basis
  (z -> z ^ mask) and whose Z part and phases drop out of |amplitude|^2.

The random draws are the reference's own (Philox stream ("trajectory", t):
``fire`` then ``codes``), so trajectory t here is trajectory t there.  For
n below the tile size all trajectories run in one launch, one CTA each
(``lrq_noisy_batch``); above it each trajectory is one fused engine run with
per-qubit mixer signs (``lrq_run_ex``) and the X string applied to the state
(``lrq_permute_xor``).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .circuit import CircuitIR, complete_edge_pairs
from .engine import Precision, ShotSet, _seam_apply, check_memory, expected_r_from_probs
from .errors import FitError, ValidationError
from .problem import WmcInstance
from .rng import derive_rng

_PAULI_BRANCH = 15.0 / 16.0


@dataclass(frozen=True)
class DepolarizingConfig:
    """Channel strength, trajectory count, and the seed all streams derive from."""

    epsilon: float
    trajectories: int = 1
    rng_seed: int = 0

    def __post_init__(self) -> None:
        if not 0.0 <= self.epsilon <= 1.0:
            raise ValidationError(f"epsilon must lie in [0, 1], got {self.epsilon}")
        if self.trajectories < 1:
            raise ValidationError(f"need at least one trajectory, got {self.trajectories}")


def epsilon_accumulated(n_2q: int, epsilon: float) -> float:
    """Total accumulated error of a circuit: two-qubit gate count times epsilon."""
    return n_2q * epsilon


# ---------------------------------------------------------------------------
# trajectories -> circuits


def _layers(circuit: CircuitIR):
    """The H^n + p x (RZZ*, RX^n) structure as per-layer gate lists."""
    n = circuit.num_qubits
    gates = circuit.gates
    if n < 2 or len(gates) < n or sorted(g.qubits[0] for g in gates[:n] if g.kind == "H") != list(range(n)):
        raise ValidationError("circuit must start with one H on every qubit")
    layers, i = [], n
    while i < len(gates):
        rzz = []
        while i < len(gates) and gates[i].kind == "RZZ":
            rzz.append(gates[i])
            i += 1
        rx = gates[i:i + n]
        if len(rx) != n or any(g.kind != "RX" for g in rx) or sorted(g.qubits[0] for g in rx) != list(range(n)):
            raise ValidationError("each layer must be RZZ gates followed by one RX on every qubit")
        layers.append((rzz, rx))
        i += n
    if not layers:
        raise ValidationError("circuit has no QAOA layer")
    return layers


def trajectory_program(circuit: CircuitIR, cfg: DepolarizingConfig, trajectory: int):
    """(phase (p, E), per-qubit mixer half-angles (p, n), final X mask) of one
    trajectory, with the reference's draws (noise.py:114-131)."""
    n = circuit.num_qubits
    layers = _layers(circuit)
    index = {pair: e for e, pair in enumerate(complete_edge_pairs(n))}
    n_rzz = sum(len(rzz) for rzz, _ in layers)
    fire = codes = None
    if cfg.epsilon > 0.0:
        rng = derive_rng(cfg.rng_seed, "trajectory", trajectory)
        fire = rng.random(n_rzz) < _PAULI_BRANCH * cfg.epsilon
        codes = rng.integers(1, 16, size=n_rzz)
    x = [0] * n  # Pauli frame pushed to the end: X part, Z part per qubit
    z = [0] * n
    phase = np.zeros((len(layers), len(index)))
    mixer = np.zeros((len(layers), n))
    k = 0
    for li, (rzz, rx) in enumerate(layers):
        for g in rzz:
            a, b = g.qubits
            sign = -1.0 if x[a] ^ x[b] else 1.0
            phase[li, index[(min(a, b), max(a, b))]] += sign * (0.5 * g.theta)
            if fire is not None and fire[k]:
                pa, pb = divmod(int(codes[k]), 4)  # 1 X, 2 Y, 3 Z on qubits (a, b)
                for q, pc in ((a, pa), (b, pb)):
                    if pc in (1, 2):
                        x[q] ^= 1
                    if pc in (2, 3):
                        z[q] ^= 1
            k += 1
        for g in rx:
            q = g.qubits[0]
            mixer[li, q] = (-1.0 if z[q] else 1.0) * (0.5 * g.theta)
    mask = sum(bit << q for q, bit in enumerate(x))
    return phase, mixer, mask


def batch_programs(circuit: CircuitIR, cfg: DepolarizingConfig):
    """trajectory_program for every trajectory at once: the Pauli frames of
    all trajectories advance together through the gate list (numpy over the
    trajectory axis).  Returns phase (T, p, E), mixer (T, p, n), xmask (T,)."""
    n, T = circuit.num_qubits, cfg.trajectories
    layers = _layers(circuit)
    index = {pair: e for e, pair in enumerate(complete_edge_pairs(n))}
    n_rzz = sum(len(rzz) for rzz, _ in layers)
    phase = np.zeros((T, len(layers), len(index)))
    mixer = np.zeros((T, len(layers), n))
    if cfg.epsilon > 0.0:
        fire = np.empty((T, n_rzz), dtype=bool)
        codes = np.empty((T, n_rzz), dtype=np.int64)
        for t in range(T):
            rng = derive_rng(cfg.rng_seed, "trajectory", t)
            fire[t] = rng.random(n_rzz) < _PAULI_BRANCH * cfg.epsilon
            codes[t] = rng.integers(1, 16, size=n_rzz)
        # X part / Z part of each code's Pauli on the gate's first / second qubit
        pa, pb = np.divmod(np.where(fire, codes, 0), 4)
        xa, za = (pa == 1) | (pa == 2), (pa == 2) | (pa == 3)
        xb, zb = (pb == 1) | (pb == 2), (pb == 2) | (pb == 3)
    x = np.zeros((T, n), dtype=bool)
    z = np.zeros((T, n), dtype=bool)
    k = 0
    for li, (rzz, rx) in enumerate(layers):
        for g in rzz:
            a, b = g.qubits
            e = index[(min(a, b), max(a, b))]
            half = 0.5 * g.theta
            phase[:, li, e] += np.where(x[:, a] ^ x[:, b], -half, half)
            if cfg.epsilon > 0.0:
                x[:, a] ^= xa[:, k]
                z[:, a] ^= za[:, k]
                x[:, b] ^= xb[:, k]
                z[:, b] ^= zb[:, k]
            k += 1
        for g in rx:
            q = g.qubits[0]
            half = 0.5 * g.theta
            mixer[:, li, q] = np.where(z[:, q], -half, half)
    xmask = (x.astype(np.uint64) << np.arange(n, dtype=np.uint64)[None, :]).sum(axis=1).astype(np.uint32)
    return phase, mixer, xmask


# The reference's host Pauli kernels (noise.py:70-98), in place on a flat
# complex array, kept as the same private seam: each runs on the GPU as one
# exact pass (lrq_apply_gate kinds 3 X, 4 Y, 5 Z).  The batched trajectory
# engine below does not use them: it propagates Pauli frames on the host.
_PAULI_KIND = (None, 3, 4, 5)


def _x_kernel(amps: np.ndarray, q: int) -> None:
    _seam_apply(amps, [(3, q, 0, 0.0)], (q,))


def _y_kernel(amps: np.ndarray, q: int) -> None:
    _seam_apply(amps, [(4, q, 0, 0.0)], (q,))


def _z_kernel(amps: np.ndarray, q: int) -> None:
    _seam_apply(amps, [(5, q, 0, 0.0)], (q,))


def _apply_pauli_pair(amps: np.ndarray, code: int, qa: int, qb: int) -> None:
    """The two-qubit Pauli numbered 1..15 (base-4 digits a, b; 0 = I, 1 X,
    2 Y, 3 Z) on qubits (qa, qb), in one upload."""
    if not 0 < int(code) < 16:
        raise ValidationError(f"two-qubit Pauli code must be 1..15, got {code}")
    pa, pb = divmod(int(code), 4)
    ops = [(_PAULI_KIND[k], q, 0, 0.0) for k, q in ((pa, qa), (pb, qb)) if k]
    _seam_apply(amps, ops, (qa, qb))


def _tile_bits(precision: Precision) -> int:
    return 13 if precision is Precision.FP32 else 12


def _batch(circuit: CircuitIR, cfg: DepolarizingConfig, precision: Precision, memory_budget, shots: int):
    """(probs (T, 2^n) or None, indices (T, shots) or None) of every trajectory.

    n below the tile: all trajectories in one lrq_noisy_batch launch.  Larger
    n: one fused engine run per trajectory (lrq_run_ex, per-qubit mixer
    signs), the X string applied to the state (lrq_permute_xor), then
    probabilities or device draws."""
    n = circuit.num_qubits
    check_memory(n, precision, memory_budget)
    phase, mixer, xmask = batch_programs(circuit, cfg)
    us = [derive_rng(cfg.rng_seed, "shots", t).random(shots) for t in range(cfg.trajectories)] if shots else None
    if n < _tile_bits(precision):
        u = np.stack(us) if shots else None
        return _native.noisy_batch(n, precision.bytes_per_amplitude, phase, mixer, xmask, u, want_probs=not shots)
    dev = _native.DeviceState(n, precision.bytes_per_amplitude)
    probs = None if shots else np.empty((cfg.trajectories, 1 << n))
    idx = np.empty((cfg.trajectories, shots), dtype=np.uint64) if shots else None
    try:
        for t in range(cfg.trajectories):
            dev.run_ex(phase[t], mixer[t])
            dev.permute_xor(int(xmask[t]))
            if shots:
                dev.recompute()
                idx[t] = dev.sample(us[t])
            else:
                a = dev.copy_amps().astype(np.complex128)
                probs[t] = a.real ** 2 + a.imag ** 2
    finally:
        dev.close()
    return probs, idx


# ---------------------------------------------------------------------------
# public API (noise.py:134-207)


def run_noisy_ensemble(circuit: CircuitIR, cfg: DepolarizingConfig, shots_per_trajectory: int,
                       precision: Precision | str = Precision.FP32, memory_budget: int | None = None,
                       threads: int = 1) -> ShotSet:
    """Sample every trajectory (stream ("shots", t)) and pool the shots in
    trajectory order; at epsilon 0 with one trajectory this reproduces the
    noiseless ``sample``.  ``threads`` is accepted for API compatibility."""
    if shots_per_trajectory < 1:
        raise ValidationError(f"shot count must be positive, got {shots_per_trajectory}")
    precision = Precision.coerce(precision)
    _, idx = _batch(circuit, cfg, precision, memory_budget, int(shots_per_trajectory))
    return ShotSet(num_qubits=circuit.num_qubits, indices=idx.reshape(-1), rng_seed=cfg.rng_seed,
                   source=f"noisy(epsilon={cfg.epsilon:g}, trajectories={cfg.trajectories})")


def noisy_expected_probs(circuit: CircuitIR, cfg: DepolarizingConfig, precision: Precision | str = Precision.FP32,
                         memory_budget: int | None = None, threads: int = 1) -> np.ndarray:
    """Trajectory-averaged basis-state distribution (channel average)."""
    precision = Precision.coerce(precision)
    probs, _ = _batch(circuit, cfg, precision, memory_budget, 0)
    acc = np.zeros(probs.shape[1])
    for row in probs:  # trajectory order, as the reference accumulates
        acc += row
    return acc / cfg.trajectories


def noisy_expected_r(circuit: CircuitIR, inst: WmcInstance, cfg: DepolarizingConfig,
                     precision: Precision | str = Precision.FP32, memory_budget: int | None = None,
                     threads: int = 1) -> float:
    """Mean approximation ratio under noise, exact per trajectory (no shots)."""
    return expected_r_from_probs(noisy_expected_probs(circuit, cfg, precision, memory_budget), inst)


# ---------------------------------------------------------------------------
# overlap ratio and decay fit (noise.py:214-270; host arithmetic)


def r_overlap(r_qpu: float, r_random: float, r_ideal: float) -> float:
    denom = r_ideal - r_random
    if denom == 0.0:
        raise ValidationError("overlap undefined: ideal and random baselines coincide")
    return (r_qpu - r_random) / denom


@dataclass(frozen=True)
class NoiseFit:
    k0: float
    r_squared: float
    n_excluded: int
    points: tuple[tuple[float, float], ...]


def fit_k0(points) -> NoiseFit:
    """Origin-constrained least squares of -log2(r_ovl) on eps_acc; points
    with r_ovl <= 0 are excluded and counted."""
    pts = [(float(a), float(r)) for a, r in points]
    used = [(a, r) for a, r in pts if r > 0.0]
    if not used:
        raise FitError("no points with positive overlap ratio to fit")
    xs = np.array([a for a, _ in used])
    ys = -np.log2(np.array([r for _, r in used]))
    sxx = float(xs @ xs)
    if sxx == 0.0:
        raise FitError("all usable points sit at zero accumulated error")
    k0 = float(xs @ ys) / sxx
    res = ys - k0 * xs
    ss_res = float(res @ res)
    ss_tot = float(((ys - ys.mean()) ** 2).sum())
    r2 = 1.0 - ss_res / ss_tot if ss_tot > 0.0 else (1.0 if ss_res < 1e-24 else 0.0)
    return NoiseFit(k0=k0, r_squared=r2, n_excluded=len(pts) - len(used), points=tuple(used))


def predict_r_overlap(k0: float, n_2q: int, epsilon: float) -> float:
    if k0 <= 0.0:
        raise ValidationError(f"decay constant must be positive, got {k0}")
    if n_2q < 0:
        raise ValidationError(f"two-qubit gate count must be non-negative, got {n_2q}")
    if not 0.0 <= epsilon <= 1.0:
        raise ValidationError(f"epsilon must lie in [0, 1], got {epsilon}")
    return float(2.0 ** (-k0 * epsilon_accumulated(n_2q, epsilon)))


__all__ = ["DepolarizingConfig", "NoiseFit", "epsilon_accumulated", "fit_k0", "noisy_expected_probs",
           "noisy_expected_r", "predict_r_overlap", "r_overlap", "run_noisy_ensemble", "trajectory_program"]
