"""Dense state-vector engine on the GPU — drop-in for lrqbench engine.py.

``run_circuit`` keeps the reference signature (engine.py:198-202) but the state
lives in HBM: the returned ``StateVector`` owns an ``lrq_state`` of liblrq.so
and copies amplitudes to the host only when ``.amps`` is read.  The circuit is
lowered to per-layer angle arrays (``circuit.lower_circuit``) and executed by
the fused sweep kernels; there is no CPU path.

Conventions kept from the reference: qubit k is bit k of the index; no
renormalisation anywhere; probabilities are float64 |a|^2 even for complex64;
the exact r divides sum p C by C* only (engine.py:214-226); sampling is the
inverse CDF normalised by its last element (engine.py:254-263) with uniforms
from Philox("shots", 0) (engine.py:272).
"""
from __future__ import annotations

import enum
import math
import os
import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _native
from .circuit import CircuitIR, lower_circuit
from .errors import CapacityError, StateError, ValidationError
from .problem import WmcInstance, index_to_bitstring
from .rng import derive_rng

# The reference's default budget models host RAM (4 GiB).  The device state
# is bounded by HBM instead: without an explicit budget or
# LRQBENCH_MEMORY_BYTES the only limit is what the device can allocate.
DEFAULT_MEMORY_BUDGET = None


class Precision(enum.Enum):
    FP32 = "fp32"
    FP64 = "fp64"

    @classmethod
    def coerce(cls, value: "Precision | str") -> "Precision":
        if isinstance(value, cls):
            return value
        try:
            return cls(str(value).lower())
        except ValueError:
            raise ValidationError(f"unknown precision {value!r}") from None

    @property
    def dtype(self) -> np.dtype:
        return np.dtype(np.complex64 if self is Precision.FP32 else np.complex128)

    @property
    def bytes_per_amplitude(self) -> int:
        return self.dtype.itemsize


def state_bytes(num_qubits: int, precision: Precision) -> int:
    return precision.bytes_per_amplitude << num_qubits


def memory_budget_bytes(override: int | None = None) -> int | None:
    if override is not None:
        return int(override)
    env = os.environ.get("LRQBENCH_MEMORY_BYTES")
    return int(env) if env else DEFAULT_MEMORY_BUDGET


def check_memory(num_qubits: int, precision: Precision, budget: int | None = None) -> None:
    need = state_bytes(num_qubits, precision)
    limit = memory_budget_bytes(budget)
    if limit is not None and need > limit:
        raise CapacityError(
            f"statevector for {num_qubits} qubits at {precision.value} needs "
            f"{need} bytes ({need / (1 << 30):.1f} GiB), budget is {limit} bytes")


class StateVector:
    """A state vector resident in HBM (one ``lrq_state``).

    ``amps`` performs an explicit device-to-host copy (cached) — only sensible
    when 2^n amplitudes fit host memory.  Reductions (norm, exact r) and
    sampling run on the device.
    """

    def __init__(self, num_qubits: int, precision: Precision, device_state: _native.DeviceState,
                 cost_weights: np.ndarray | None = None):
        self.num_qubits = num_qubits
        self._precision = precision
        self._dev = device_state
        self._cost = None if cost_weights is None else np.asarray(cost_weights, dtype=np.float64)
        self._amps = None

    @property
    def precision(self) -> Precision:
        return self._precision

    @property
    def device_state(self) -> _native.DeviceState:
        return self._dev

    @property
    def amps(self) -> np.ndarray:
        if self._amps is None:
            self._amps = self._dev.copy_amps()
        return self._amps

    def release(self) -> None:
        """Free the device memory now (the handle is also freed on GC)."""
        self._dev.close()

    def _reductions(self, weights: np.ndarray | None):
        """Final-pass reductions for cost ``weights`` (None: any cost)."""
        if weights is not None and (self._cost is None or not np.array_equal(self._cost, weights)):
            self._dev.set_cost(weights)
            self._dev.recompute()
            self._cost = np.array(weights, dtype=np.float64)
        elif self._cost is None and weights is None:
            try:
                return self._dev.reduce()
            except StateError:
                self._dev.recompute()
        return self._dev.reduce()

    def _copy_range(self, start: int, count: int) -> np.ndarray:
        return self._dev.copy_amps(start, count)

    def _draw(self, u: np.ndarray) -> np.ndarray:
        """Global indices of the inverse-CDF draws for uniforms u."""
        self._reductions(None)
        return self._dev.sample(u)

    def norm_squared(self) -> float:
        return float(self._reductions(None).sum_p)

    def norm_tolerance(self) -> float:
        eps = np.finfo(np.float32 if self._precision is Precision.FP32 else np.float64).eps
        return 10.0 * (1 << self.num_qubits) * float(eps)

    def probabilities(self) -> np.ndarray:
        a = self.amps.astype(np.complex128, copy=False)
        return (a.real ** 2 + a.imag ** 2).astype(np.float64)


def _device_state(num_qubits: int, precision: Precision, memory_budget: int | None):
    if num_qubits < 1:
        raise ValidationError(f"need at least one qubit, got {num_qubits}")
    check_memory(num_qubits, precision, memory_budget)
    return _native.DeviceState(num_qubits, precision.bytes_per_amplitude)


_GATE_KIND = {"H": 0, "RX": 1, "RZZ": 2}


def zero_state(num_qubits: int, precision: Precision | str = Precision.FP32,
               memory_budget: int | None = None) -> StateVector:
    """|0...0> in HBM (engine.py:99-110)."""
    precision = Precision.coerce(precision)
    dev = _device_state(num_qubits, precision, memory_budget)
    dev.reset(0)
    return StateVector(num_qubits, precision, dev)


def init_plus_state(num_qubits: int, precision: Precision | str = Precision.FP32,
                    memory_budget: int | None = None) -> StateVector:
    """Uniform superposition with amplitude 2^(-n/2) (engine.py:113-121)."""
    precision = Precision.coerce(precision)
    dev = _device_state(num_qubits, precision, memory_budget)
    dev.reset(1)
    return StateVector(num_qubits, precision, dev)


def _touch(sv: StateVector) -> None:
    sv._amps = None  # host copy and reductions are stale after a gate
    sv._cost = None


def apply_h(sv: StateVector, q: int) -> None:
    sv.device_state.apply_gate(0, q)
    _touch(sv)


def apply_rx(sv: StateVector, theta: float, q: int) -> None:
    sv.device_state.apply_gate(1, q, 0, theta)
    _touch(sv)


def apply_rzz(sv: StateVector, theta: float, qa: int, qb: int) -> None:
    sv.device_state.apply_gate(2, qa, qb, theta)
    _touch(sv)


def apply_gate(sv: StateVector, gate) -> None:
    """One gate, one pass over the state on the GPU (engine.py:158-195)."""
    q1 = gate.qubits[1] if len(gate.qubits) > 1 else 0
    sv.device_state.apply_gate(_GATE_KIND[gate.kind], gate.qubits[0], q1, gate.theta or 0.0)
    _touch(sv)


def run_circuit(circuit: CircuitIR, precision: Precision | str = Precision.FP32,
                memory_budget: int | None = None) -> StateVector:
    """Evolve |0...0> through the circuit on the GPU.

    H + p x (RZZ block, RX^n) circuits (everything build_circuit makes) run as
    fused sweeps; any other gate list runs gate by gate (engine.py:198-207)."""
    precision = Precision.coerce(precision)
    check_memory(circuit.num_qubits, precision, memory_budget)
    try:
        layers = lower_circuit(circuit)
    except ValidationError:
        sv = zero_state(circuit.num_qubits, precision, memory_budget)
        for g in circuit.gates:
            apply_gate(sv, g)
        return sv
    dev = _device_state(circuit.num_qubits, precision, memory_budget)
    cost = getattr(circuit, "cost_weights", None)
    if cost is not None:
        dev.set_cost(cost)
    dev.run(layers.phase, layers.mixer)
    return StateVector(circuit.num_qubits, precision, dev, cost)


# ---------------------------------------------------------------------------
# observables and sampling


_EXPECTATION_CHUNK = 1 << 16


def expected_r_from_probs(probs: np.ndarray, inst: WmcInstance) -> float:
    """Expected approximation ratio of an explicit basis-state distribution
    (engine.py:214-226): chunked probs . C / C*, cut values from the GPU."""
    from .problem import cut_values_range

    probs = np.asarray(probs, dtype=np.float64)
    if probs.size != 1 << inst.num_vertices:
        raise ValidationError(f"distribution over {probs.size} states does not match n={inst.num_vertices}")
    if inst.optimal_cut is None:
        raise StateError("instance has no optimal cut; solve it first")
    total = 0.0
    for lo in range(0, probs.size, _EXPECTATION_CHUNK):
        hi = min(lo + _EXPECTATION_CHUNK, probs.size)
        total += float(probs[lo:hi] @ cut_values_range(inst, lo, hi))
    return total / inst.optimal_cut.value


def exact_expected_r(sv: StateVector, inst: WmcInstance) -> float:
    """sum_z |a_z|^2 C(z) / C* over the full distribution (no sampling)."""
    if inst.num_vertices != sv.num_qubits:
        raise ValidationError(
            f"instance has {inst.num_vertices} vertices, state has {sv.num_qubits} qubits")
    if inst.optimal_cut is None:
        raise StateError("instance has no optimal cut; solve it first")
    red = sv._reductions(inst.weights())
    return float(red.sum_p_cut) / inst.optimal_cut.value


@dataclass(eq=False)
class ShotSet:
    num_qubits: int
    indices: np.ndarray
    rng_seed: int | None
    source: str

    def __len__(self) -> int:
        return int(self.indices.size)

    def bitstrings(self) -> list[str]:
        return [index_to_bitstring(int(z), self.num_qubits) for z in self.indices]


def sample(sv: StateVector, n_shots: int, rng_seed: int) -> ShotSet:
    """Inverse-CDF draws over |a|^2 with uniforms from Philox("shots", 0)."""
    if n_shots < 1:
        raise ValidationError(f"shot count must be positive, got {n_shots}")
    u = derive_rng(rng_seed, "shots", 0).random(n_shots)
    return ShotSet(sv.num_qubits, sv._draw(u), int(rng_seed), "noiseless")


# ---------------------------------------------------------------------------
# LQSV dump (engine.py:279-312 format: "<4sBBH" header + little-endian re/im)

_MAGIC = b"LQSV"
_HEADER = struct.Struct("<4sBBH")


def save_statevector(sv: StateVector, path: str | Path) -> None:
    fbytes = sv.precision.bytes_per_amplitude // 2
    code = "<c8" if sv.precision is Precision.FP32 else "<c16"
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(_MAGIC, 1, fbytes, sv.num_qubits))
        chunk = 1 << 24
        total = 1 << sv.num_qubits
        for lo in range(0, total, chunk):
            part = sv._copy_range(lo, min(chunk, total - lo))
            fh.write(np.ascontiguousarray(part, dtype=code).tobytes())


def load_statevector(path: str | Path, memory_budget: int | None = None) -> StateVector:
    """LQSV dump -> a state in HBM (engine.py:296-312), streamed in chunks."""
    raw = Path(path).read_bytes()
    if len(raw) < _HEADER.size:
        raise ValidationError(f"{path} is not a statevector dump (truncated header)")
    magic, version, fbytes, n = _HEADER.unpack_from(raw)
    if magic != _MAGIC or version != 1:
        raise ValidationError(f"{path} is not a statevector dump (bad magic/version)")
    if fbytes not in (4, 8):
        raise ValidationError(f"{path} has unsupported float width {fbytes}")
    precision = Precision.FP32 if fbytes == 4 else Precision.FP64
    code = "<c8" if fbytes == 4 else "<c16"
    amps = np.frombuffer(raw, dtype=code, offset=_HEADER.size)
    if amps.size != 1 << n:
        raise ValidationError(f"{path} payload has {amps.size} amplitudes, expected {1 << n}")
    dev = _device_state(n, precision, memory_budget)
    chunk = 1 << 24
    for lo in range(0, amps.size, chunk):
        dev.store_amps(amps[lo:lo + chunk], lo)
    return StateVector(n, precision, dev)


def load_statevector_amps(path: str | Path) -> tuple[int, np.ndarray]:
    """Read an LQSV dump into host memory: (num_qubits, amplitudes)."""
    raw = Path(path).read_bytes()
    if len(raw) < _HEADER.size:
        raise ValidationError(f"{path} is not a statevector dump (truncated header)")
    magic, version, fbytes, n = _HEADER.unpack_from(raw)
    if magic != _MAGIC or version != 1:
        raise ValidationError(f"{path} is not a statevector dump (bad magic/version)")
    if fbytes not in (4, 8):
        raise ValidationError(f"{path} has unsupported float width {fbytes}")
    code = "<c8" if fbytes == 4 else "<c16"
    amps = np.frombuffer(raw, dtype=code, offset=_HEADER.size)
    if amps.size != 1 << n:
        raise ValidationError(f"{path} payload has {amps.size} amplitudes, expected {1 << n}")
    return n, amps.astype(np.complex64 if fbytes == 4 else np.complex128)


def uniform_amplitude(num_qubits: int, precision: Precision | str) -> complex:
    """Value of every amplitude after the H layer (sequential products)."""
    precision = Precision.coerce(precision)
    t = np.float32 if precision is Precision.FP32 else np.float64
    r = t(1.0 / math.sqrt(2.0))
    v = t(1.0)
    for _ in range(num_qubits):
        v = t(v * r)
    return complex(v)
