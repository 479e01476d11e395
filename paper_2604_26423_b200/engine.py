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

# The reference's default budget (engine.py:31): 4 GiB unless
# LRQBENCH_MEMORY_BYTES or an explicit memory_budget says otherwise.  The
# same contract holds here, so a drop-in user sees the same CapacityError;
# large device states pass a budget (bench.py, the CLI's --memory-bytes).
DEFAULT_MEMORY_BUDGET = 4 << 30


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


def drain_state_pool() -> None:
    """Free the HBM of dropped states kept for reuse.  A dropped StateVector's
    allocation is parked for the next state of the same shape (no cudaMalloc
    per run_circuit); this library's own allocations drain the pool when they
    run out, other code that needs the memory calls this first.
    StateVector.release() frees a state at once."""
    _native.drain_pool()


def state_bytes(num_qubits: int, precision: Precision) -> int:
    return precision.bytes_per_amplitude << num_qubits


def memory_budget_bytes(override: int | None = None) -> int:
    if override is not None:
        return int(override)
    return int(os.environ.get("LRQBENCH_MEMORY_BYTES", DEFAULT_MEMORY_BUDGET))


def check_memory(num_qubits: int, precision: Precision, budget: int | None = None) -> None:
    need = state_bytes(num_qubits, precision)
    limit = memory_budget_bytes(budget)
    if need > limit:
        raise CapacityError(
            f"statevector for {num_qubits} qubits at {precision.value} needs "
            f"{need} bytes ({need / (1 << 30):.1f} GiB), budget is {limit} bytes")


class StateVector:
    """A state vector resident in HBM (one ``lrq_state``).

    Two constructions: the reference's ``StateVector(num_qubits, amps)``
    (engine.py:77-96) uploads a host array (complex64 stays FP32, anything
    else becomes complex128 / FP64); the engine wraps a device state it made
    (``StateVector._wrap``).  ``amps`` is an explicit device-to-host copy,
    cached and read-only (a write to it would not reach the device, so it
    raises instead of being dropped); gates and runs invalidate the cache.
    Reductions (norm, exact r) and sampling run on the device.
    """

    def __init__(self, num_qubits: int, amps=None, *, device_state: "_native.DeviceState | None" = None,
                 precision: "Precision | None" = None, cost_weights: np.ndarray | None = None):
        self.num_qubits = int(num_qubits)
        self._cost = None if cost_weights is None else np.asarray(cost_weights, dtype=np.float64)
        self._amps = None
        if device_state is None:
            if amps is None:
                raise ValidationError("StateVector needs amplitudes (or a device state)")
            a = np.asarray(amps)
            a = a if a.dtype == np.complex64 else a.astype(np.complex128)
            if a.ndim != 1 or a.size != 1 << self.num_qubits:
                raise ValidationError(f"{a.size} amplitudes do not form a {self.num_qubits}-qubit state")
            precision = Precision.FP32 if a.dtype == np.complex64 else Precision.FP64
            device_state = _native.DeviceState(self.num_qubits, precision.bytes_per_amplitude)
            device_state.store_amps(a)
        elif precision is None:
            precision = Precision.FP32 if device_state.precision_bytes == 8 else Precision.FP64
        self._precision = precision
        self._dev = device_state

    @classmethod
    def _wrap(cls, num_qubits: int, precision: Precision, device_state: "_native.DeviceState",
              cost_weights: np.ndarray | None = None) -> "StateVector":
        return cls(num_qubits, device_state=device_state, precision=precision, cost_weights=cost_weights)

    @property
    def precision(self) -> Precision:
        return self._precision

    @property
    def device_state(self) -> _native.DeviceState:
        if self._dev is None:
            raise StateError("state vector has been released")
        return self._dev

    @property
    def amps(self) -> np.ndarray:
        if self._amps is None:
            a = self.device_state.copy_amps()
            a.setflags(write=False)
            self._amps = a
        return self._amps

    def release(self) -> None:
        """Free the device memory now (cudaFree; not parked for reuse)."""
        if self._dev is not None:
            self._dev.close(park=False)
            self._dev = None
        self._amps = None

    def _reductions(self, weights: np.ndarray | None):
        """Final-pass reductions for cost ``weights`` (None: any cost)."""
        dev = self.device_state
        if weights is not None and (self._cost is None or not np.array_equal(self._cost, weights)):
            dev.set_cost(weights)
            dev.recompute()
            self._cost = np.array(weights, dtype=np.float64)
        elif self._cost is None and weights is None:
            try:
                return dev.reduce()
            except StateError:
                dev.recompute()
        return dev.reduce()

    def _copy_range(self, start: int, count: int) -> np.ndarray:
        return self.device_state.copy_amps(start, count)

    def _draw(self, u: np.ndarray) -> np.ndarray:
        """Global indices of the inverse-CDF draws for uniforms u."""
        self._reductions(None)
        return self.device_state.sample(u)

    def norm_squared(self) -> float:
        return float(self._reductions(None).sum_p)

    def norm_tolerance(self) -> float:
        eps = np.finfo(np.float32 if self._precision is Precision.FP32 else np.float64).eps
        return 10.0 * (1 << self.num_qubits) * float(eps)

    def probabilities(self) -> np.ndarray:
        a = self.amps.astype(np.complex128, copy=False)
        return (a.real ** 2 + a.imag ** 2).astype(np.float64)

    def _histogram(self, weights: np.ndarray, bins: int, lo: float, hi: float):
        """One read-only pass with the E histogram on: (raw bins, reductions)."""
        dev = self.device_state
        dev.set_cost(weights)
        dev.set_search(True)  # the extremes of C come from the same pass
        dev.set_histogram(bins, lo, hi)
        try:
            dev.recompute()
            raw = dev.histogram()
            red = dev.reduce()
        finally:
            dev.set_histogram(0)
        self._cost = np.array(weights, dtype=np.float64)
        return raw, red


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
    return StateVector._wrap(num_qubits, precision, dev)


def init_plus_state(num_qubits: int, precision: Precision | str = Precision.FP32,
                    memory_budget: int | None = None) -> StateVector:
    """Uniform superposition with amplitude 2^(-n/2) (engine.py:113-121)."""
    precision = Precision.coerce(precision)
    dev = _device_state(num_qubits, precision, memory_budget)
    dev.reset(1)
    return StateVector._wrap(num_qubits, precision, dev)


def _touch(sv: StateVector) -> None:
    sv._amps = None  # host copy and reductions are stale after a gate
    sv._cost = None


def _check_qubit(sv: StateVector, q: int) -> None:
    if not 0 <= q < sv.num_qubits:
        raise ValidationError(f"qubit {q} out of range for {sv.num_qubits} qubits")


def apply_h(sv: StateVector, q: int) -> None:
    _check_qubit(sv, q)
    sv.device_state.apply_gate(0, q)
    _touch(sv)


def apply_rx(sv: StateVector, theta: float, q: int) -> None:
    _check_qubit(sv, q)
    sv.device_state.apply_gate(1, q, 0, theta)
    _touch(sv)


def apply_rzz(sv: StateVector, theta: float, qa: int, qb: int) -> None:
    _check_qubit(sv, qa)
    _check_qubit(sv, qb)
    if qa == qb:
        raise ValidationError("RZZ qubits must differ")
    sv.device_state.apply_gate(2, qa, qb, theta)
    _touch(sv)


def apply_gate(sv: StateVector, gate) -> None:
    """One gate, one pass over the state on the GPU (engine.py:158-195)."""
    for q in gate.qubits:
        _check_qubit(sv, q)
    q1 = gate.qubits[1] if len(gate.qubits) > 1 else 0
    sv.device_state.apply_gate(_GATE_KIND[gate.kind], gate.qubits[0], q1, gate.theta or 0.0)
    _touch(sv)


# scratch device states of the per-gate seam, one per (n, precision)
_SEAM: dict = {}


def _apply_gate_kernel(amps: np.ndarray, gate, qubits: tuple) -> None:
    """The reference's per-gate seam (engine.py:158-166) on the GPU: the
    host array is uploaded, the gate runs as one device pass (the same
    gate kernels as apply_gate), and the result is written back in place.
    Callers that own device states use apply_gate instead; this keeps code
    written against the reference's raw-array kernels working."""
    if gate.kind not in _GATE_KIND:
        raise ValidationError(f"unknown gate kind {gate.kind!r}")
    q1 = qubits[1] if len(qubits) > 1 else 0
    _seam_apply(amps, [(_GATE_KIND[gate.kind], qubits[0], q1, gate.theta or 0.0)], qubits)


def _seam_apply(amps: np.ndarray, ops, qubits) -> None:
    """Host-array seam: upload, run `ops` ((kind, q0, q1, theta): lrq_apply_gate
    kinds 0 H, 1 RX, 2 RZZ, 3 X, 4 Y, 5 Z) as device passes, write back in place."""
    if amps.dtype not in (np.complex64, np.complex128) or amps.ndim != 1:
        raise ValidationError("the gate seam works on a flat complex64/complex128 array")
    n = amps.size.bit_length() - 1
    if amps.size != 1 << n:
        raise ValidationError(f"{amps.size} amplitudes do not form a state vector")
    for q in qubits:
        if not 0 <= q < n:
            raise ValidationError(f"qubit {q} out of range for {n} qubits")
    if not ops:
        return
    pb = amps.dtype.itemsize
    dev = _SEAM.get((n, pb))
    if dev is None:
        dev = _SEAM[(n, pb)] = _native.DeviceState(n, pb)
    dev.store_amps(amps)
    for kind, q0, q1, theta in ops:
        dev.apply_gate(kind, q0, q1, theta)
    amps[...] = dev.copy_amps()


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
    # a solved instance's C* is known: the final pass only sums p and p*C
    dev.set_search(getattr(circuit, "cost_optimum", None) is None)
    dev.run(layers.phase, layers.mixer)
    return StateVector._wrap(circuit.num_qubits, precision, dev, cost)


# ---------------------------------------------------------------------------
# observables and sampling


_EXPECTATION_CHUNK = 1 << 16


def expected_r_from_probs(probs: np.ndarray, inst: WmcInstance) -> float:
    """Expected approximation ratio of an explicit basis-state distribution
    (engine.py:214-226): sum over 2^16 chunks of probs . C_spin / C*, in one
    device call (lrq_expected_cut); the chunk sums are added in order."""
    probs = np.asarray(probs, dtype=np.float64)
    if probs.size != 1 << inst.num_vertices:
        raise ValidationError(f"distribution over {probs.size} states does not match n={inst.num_vertices}")
    if inst.optimal_cut is None:
        raise StateError("instance has no optimal cut; solve it first")
    chunks = _native.expected_cut_chunks(inst.num_vertices, inst.weights(), 0.5 * inst.total_weight(), probs)
    total = 0.0
    for c in chunks:
        total += float(c)
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


@dataclass
class CutDistribution:
    """Exact distribution of the cut value C under |psi|^2, binned on the
    device by the fused final pass (lrq_set_histogram): probs[b] is the total
    probability of the basis states with C in [edges[b], edges[b+1]).  Plus
    the pass's extremes: min/max of C over all basis states (C = (W - E)/2)."""
    edges: np.ndarray
    probs: np.ndarray
    cut_min: float
    cut_max: float

    def bin_of(self, cuts: np.ndarray) -> np.ndarray:
        b = np.searchsorted(self.edges, np.asarray(cuts, dtype=np.float64), side="right") - 1
        return np.clip(b, 0, self.probs.size - 1)


def exact_cut_distribution(sv, inst: WmcInstance, bins: int = 2048) -> CutDistribution:
    """The exact C distribution of a state (any engine: dense, sharded,
    distributed - collective there), from one read-only device pass over the
    state with the histogram on (chi-square reference of the
    sampled shots at sizes where |psi|^2 never leaves the device)."""
    if inst.num_vertices != sv.num_qubits:
        raise ValidationError(f"instance has {inst.num_vertices} vertices, state has {sv.num_qubits} qubits")
    if not 1 <= bins <= 4096:
        raise ValidationError(f"bins must be in [1, 4096], got {bins}")
    w = inst.weights()
    W = float(np.sum(np.abs(w)))
    lo, hi = -W * (1 + 1e-12) - 1e-12, W * (1 + 1e-12) + 1e-12  # E in [-W, W]
    raw, red = sv._histogram(w, bins, lo, hi)
    probs = raw.astype(np.float64) / float(1 << 60)
    e_edges = np.linspace(lo, hi, bins + 1)
    # C = (W_tot - E) / 2 is decreasing in E: reverse to ascending C
    wt = inst.total_weight()
    c_edges = ((wt - e_edges) / 2.0)[::-1]
    return CutDistribution(c_edges, probs[::-1].copy(), 0.5 * (wt - red.max_energy), 0.5 * (wt - red.min_energy))


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


def draw_indices(probs: np.ndarray, n_shots: int, rng: np.random.Generator) -> np.ndarray:
    """Inverse-CDF draw over an unnormalised float64 distribution
    (engine.py:254-263) on the GPU (lrq_draw_indices): the uniforms come from
    ``rng`` on the host, the CDF search runs on the device."""
    if n_shots < 1:
        raise ValidationError(f"shot count must be positive, got {n_shots}")
    probs = np.asarray(probs, dtype=np.float64).ravel()
    if probs.size == 0:
        raise ValidationError("statevector has zero norm, nothing to sample")
    return _native.draw_indices(probs, rng.random(n_shots))


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


_DUMP_CHUNK = 1 << 24  # amplitudes per host round trip of a streamed dump / load


def lqsv_header(path: str | Path) -> tuple[int, "Precision", int]:
    """(num_qubits, precision, payload offset) of an LQSV dump, validated
    like the reference's loader (engine.py:296-312) without reading the payload."""
    p = Path(path)
    size = p.stat().st_size if p.exists() else 0
    with open(p, "rb") as fh:
        head = fh.read(_HEADER.size)
    if len(head) < _HEADER.size:
        raise ValidationError(f"{path} is not a statevector dump (truncated header)")
    magic, version, fbytes, n = _HEADER.unpack_from(head)
    if magic != _MAGIC or version != 1:
        raise ValidationError(f"{path} is not a statevector dump (bad magic/version)")
    if fbytes not in (4, 8):
        raise ValidationError(f"{path} has unsupported float width {fbytes}")
    precision = Precision.FP32 if fbytes == 4 else Precision.FP64
    want = _HEADER.size + (precision.bytes_per_amplitude << n)
    if size != want:
        amps = (size - _HEADER.size) // precision.bytes_per_amplitude
        raise ValidationError(f"{path} payload has {amps} amplitudes, expected {1 << n}")
    return n, precision, _HEADER.size


def lqsv_create(path: str | Path, num_qubits: int, precision: "Precision") -> None:
    """Write the header and size the file: ranks / shards then fill their
    own byte ranges (lqsv_write_range) in any order, concurrently."""
    fbytes = precision.bytes_per_amplitude // 2
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(_MAGIC, 1, fbytes, num_qubits))
        fh.truncate(_HEADER.size + (precision.bytes_per_amplitude << num_qubits))


def lqsv_write_range(path: str | Path, dev, global_start: int, count: int, precision: "Precision") -> None:
    """Stream the local amplitudes [0, count) of device state `dev` into the
    dump at global index global_start (little-endian re/im, chunked D2H)."""
    code = "<c8" if precision is Precision.FP32 else "<c16"
    B = precision.bytes_per_amplitude
    with open(path, "r+b") as fh:
        fh.seek(_HEADER.size + global_start * B)
        for lo in range(0, count, _DUMP_CHUNK):
            part = dev.copy_amps(lo, min(_DUMP_CHUNK, count - lo))
            fh.write(np.ascontiguousarray(part, dtype=code).tobytes())


def lqsv_read_range(path: str | Path, dev, global_start: int, count: int, precision: "Precision") -> None:
    """Stream the dump's amplitudes [global_start, +count) into the local
    amplitudes [0, count) of device state `dev` (chunked H2D)."""
    code = "<c8" if precision is Precision.FP32 else "<c16"
    B = precision.bytes_per_amplitude
    with open(path, "rb") as fh:
        fh.seek(_HEADER.size + global_start * B)
        for lo in range(0, count, _DUMP_CHUNK):
            m = min(_DUMP_CHUNK, count - lo)
            dev.store_amps(np.frombuffer(fh.read(m * B), dtype=code), lo)


def save_statevector(sv, path: str | Path) -> None:
    """LQSV dump (engine.py:279-293 format) streamed from the device in
    chunks; a sharded state writes every shard's range from its own thread
    (sharded.ShardedStateVector.save), a distributed one from every rank
    (distributed.DistStateVector.save)."""
    if hasattr(sv, "save"):
        sv.save(path)
        return
    lqsv_create(path, sv.num_qubits, sv.precision)
    lqsv_write_range(path, sv.device_state, 0, 1 << sv.num_qubits, sv.precision)


def load_statevector(path: str | Path, memory_budget: int | None = None) -> StateVector:
    """LQSV dump -> a state in HBM (engine.py:296-312), streamed in chunks."""
    n, precision, _ = lqsv_header(path)
    dev = _device_state(n, precision, memory_budget)
    lqsv_read_range(path, dev, 0, 1 << n, precision)
    return StateVector._wrap(n, precision, dev)


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
