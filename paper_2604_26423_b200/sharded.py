"""Sharded execution — drop-in for lrqbench sharded.py.

The reference (sharded.py:1-21, 200-385) splits the amplitude array into
2^(nq - nq_local) shards owned by one host thread each and runs the gate list
gate by gate; every gate on a global qubit swaps half a shard with a partner
shard, applies the gate, and swaps back.

Here a shard is an ``lrq_state`` of an in-process shard group (``lrq_group``,
include/lrq.h): one host thread per shard makes the engine's collective calls
(the same ones the one-process-per-GPU NCCL engine makes), the shards sit on
the visible devices (several shards may share one), and the circuit runs as
the distributed sweep plan: the cost phase is local to every
shard, and the mixer of the global qubits costs one block-transpose remap per
layer instead of two half-shard swaps per global gate.

Kept from the reference: the plan types and their validation, the static
per-gate exchange accounting (``exchange_steps`` / ``exchange_volume``), the
timing record and CSV schema, the scaling sweeps, and "a worker failure
aborts the run" (``AbortedRunError``).  Different by design:

* ``TimingRecord.gates`` has one row per device launch of the sweep plan
  (kind = sweep letter, see ``LAUNCH_KINDS``), not one per gate;
  ``amps_exchanged`` counts what the remaps moved (``remap_volume``);
* sharded and dense amplitudes agree to rounding (1e-12 relative in
  complex128), not bit for bit: the sharded plan applies the mixer qubits in
  a different order;
* shards smaller than the engine's tile (2^(12+g) complex128 /
  2^(13+g) complex64 amplitudes in total) are run as one dense state.
"""
from __future__ import annotations

import csv
import json
import threading
import time
from dataclasses import dataclass, field
from typing import IO, Callable, Iterable

import numpy as np

from . import _native
from .circuit import CircuitIR, GateOp, LrQaoaParams, build_circuit, lower_circuit
from .engine import Precision, StateVector, _device_state, check_memory
from .errors import AbortedRunError, ValidationError
from .problem import generate_instance

# sweep-plan launch kinds reported in TimingRecord rows
LAUNCH_KINDS = {
    "P": "prepare+mix",   # H layer, phase_1, mixer_1 on the first qubit group
    "M": "mix",           # mixer on one qubit group
    "F": "mix+phase+mix",  # mixer_k, phase_{k+1}, mixer_{k+1} fused
    "R": "mix+reduce",    # last mixer + final reductions
    "L": "mix (partial)",
    "Q": "reduce",        # read-only final pass
    "N": "search",
    "T": "remap",         # block-transpose exchange of the global qubits
    "Y": "remap (fused)",  # the preceding sweep stored into the peers' buffers; barrier
    "W": "remap (pipelined)",  # the preceding sweep ran block by block, swaps overlapped; tail wait
    "X": "flip",          # deferred global X: index reversal + mirror exchange
    "S": "small",
    "Z": "finalize",
}


# ---------------------------------------------------------------------------
# plans (sharded.py:43-73)


@dataclass(frozen=True)
class ShardPlan:
    nq: int
    nq_local: int
    num_shards: int
    shard_len: int


def plan_shards(nq: int, nq_local: int) -> ShardPlan:
    """Split nq qubits into 2^(nq - nq_local) shards of 2^nq_local amplitudes."""
    if nq < 1:
        raise ValidationError(f"need at least one qubit, got {nq}")
    if not 1 <= nq_local <= nq:
        raise ValidationError(f"nq_local must satisfy 1 <= nq_local <= nq, got {nq_local} for nq={nq}")
    return ShardPlan(nq=nq, nq_local=nq_local, num_shards=1 << (nq - nq_local), shard_len=1 << nq_local)


def plan_for_shard_count(nq: int, num_shards: int) -> ShardPlan:
    if num_shards < 1 or num_shards & (num_shards - 1):
        raise ValidationError(f"shard count must be a power of two, got {num_shards}")
    g = num_shards.bit_length() - 1
    if g >= nq:
        raise ValidationError(f"{num_shards} shards need more than {nq} qubits")
    return plan_shards(nq, nq - g)


# ---------------------------------------------------------------------------
# the reference's per-gate exchange accounting (sharded.py:76-130)


@dataclass(frozen=True)
class ExchangeStep:
    """One pairwise half-block swap of the reference engine."""

    global_qubit: int
    local_slot: int
    pair_bit: int
    amps_per_shard: int

    def partner(self, shard: int) -> int:
        return shard ^ (1 << self.pair_bit)

    def pairs(self, num_shards: int) -> list[tuple[int, int]]:
        return [(s, s ^ (1 << self.pair_bit)) for s in range(num_shards) if not (s >> self.pair_bit) & 1]


def exchange_steps(gate: GateOp, plan: ShardPlan) -> list[ExchangeStep]:
    """Steps the reference needs for one gate: its global qubits (highest
    first) paired with spare local slots taken from the top of the shard,
    skipping the gate's own local qubits."""
    glob = sorted((q for q in gate.qubits if q >= plan.nq_local), reverse=True)
    if not glob:
        return []
    busy = {q for q in gate.qubits if q < plan.nq_local}
    free = [q for q in range(plan.nq_local - 1, -1, -1) if q not in busy]
    if len(free) < len(glob):
        raise ValidationError(f"shards of 2^{plan.nq_local} amplitudes cannot host gate on {gate.qubits}")
    return [ExchangeStep(global_qubit=q, local_slot=slot, pair_bit=q - plan.nq_local,
                         amps_per_shard=plan.shard_len // 2) for q, slot in zip(glob, free)]


def exchange_volume(circuit: CircuitIR, plan: ShardPlan) -> int:
    """Amplitudes the reference's per-gate swaps would move over the run."""
    per = plan.num_shards * (plan.shard_len // 2)
    return sum(len(exchange_steps(g, plan)) for g in circuit.gates) * per


def _engine_shards(nq: int, num_shards: int, precision: Precision, p: int) -> bool:
    """True if the tile engine runs this plan as real shards."""
    if num_shards < 2:
        return False
    try:
        _native.describe_dist_plan(nq, num_shards.bit_length() - 1, precision.bytes_per_amplitude, p)
    except ValidationError:
        return False
    return True


def _flips(mixer: np.ndarray) -> int:
    """Layers whose RX takes the deferred-X form (|sin h| > |cos h|, mixer_form)."""
    return int(np.sum(np.abs(np.sin(mixer)) > np.abs(np.cos(mixer))))


def remap_volume(circuit: CircuitIR, plan: ShardPlan, precision: Precision | str = Precision.FP32) -> int:
    """Amplitudes this engine moves between shards over the run: one block
    transpose per layer ((G-1)/G of the state) and a full mirror exchange
    when an odd number of layers took the deferred-X mixer form.  (An odd p
    leaves the state in the swapped layout; reading its amplitudes makes one
    more transpose then, lrq_restore_layout.)"""
    precision = Precision.coerce(precision)
    layers = lower_circuit(circuit)
    p = int(layers.mixer.size)
    G = plan.num_shards
    if not _engine_shards(plan.nq, G, precision, p):
        return 0
    plan_js = json.loads(_native.describe_dist_plan(plan.nq, G.bit_length() - 1, precision.bytes_per_amplitude, p))
    remaps = sum(int(r) for _, r, _ in plan_js["dist"])
    vol = remaps * ((G - 1) << (plan.nq - (G.bit_length() - 1)))
    if _flips(layers.mixer) & 1:
        vol += 1 << plan.nq
    return vol


# ---------------------------------------------------------------------------
# timing (sharded.py:133-195)


@dataclass(frozen=True)
class GateTiming:
    gate_index: int
    kind: str
    compute_s: float
    exchange_s: float
    amps_exchanged: int


@dataclass
class TimingRecord:
    nq: int
    p: int
    num_shards: int
    wall_seconds: float
    gates: list[GateTiming] = field(default_factory=list)

    @property
    def compute_seconds(self) -> float:
        return sum(g.compute_s for g in self.gates)

    @property
    def exchange_seconds(self) -> float:
        return sum(g.exchange_s for g in self.gates)

    @property
    def amps_exchanged(self) -> int:
        return sum(g.amps_exchanged for g in self.gates)


TIMING_CSV_FIELDS = ("nq", "p", "num_shards", "gate_index", "kind", "compute_s", "exchange_s", "amps_exchanged")


def write_timing_csv(records: Iterable[TimingRecord], fh: IO[str]) -> None:
    w = csv.writer(fh)
    w.writerow(TIMING_CSV_FIELDS)
    for rec in records:
        for g in rec.gates:
            w.writerow([rec.nq, rec.p, rec.num_shards, g.gate_index, g.kind, f"{g.compute_s:.9f}",
                        f"{g.exchange_s:.9f}", g.amps_exchanged])


# ---------------------------------------------------------------------------
# the sharded state


def _collective(group: _native.ShardGroup, shards: list, fn: Callable) -> list:
    """Run fn(rank, shard) on one host thread per shard (ctypes drops the GIL
    inside the engine).  Any failure aborts the group and the run."""
    out = [None] * len(shards)
    errs: list[BaseException] = []

    def body(r):
        try:
            out[r] = fn(r, shards[r])
        except BaseException as exc:  # noqa: BLE001 - surfaced below
            errs.append(exc)
            try:
                group.abort()
            except Exception:
                pass

    threads = [threading.Thread(target=body, args=(r,), name=f"shard-{r}", daemon=True) for r in range(len(shards))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errs:
        raise AbortedRunError(f"shard worker failed: {errs[0]}") from errs[0]
    return out


class ShardedStateVector:
    """A state held as G shard states (shard s = amplitudes whose top g bits
    equal s).  Same read interface as ``engine.StateVector``."""

    def __init__(self, plan: ShardPlan, precision: Precision, group: _native.ShardGroup, shards: list,
                 cost_weights: np.ndarray | None):
        self.num_qubits = plan.nq
        self.plan = plan
        self._precision = precision
        self._group = group
        self._shards = shards
        self._cost = None if cost_weights is None else np.asarray(cost_weights, dtype=np.float64)
        self._amps = None

    @property
    def precision(self) -> Precision:
        return self._precision

    @property
    def num_shards(self) -> int:
        return len(self._shards)

    def _identity_layout(self) -> None:
        """An odd-p run leaves the shards in the swapped layout (the final
        pass ran there); amplitude reads need the remaining remap first."""
        if any(s.layout() for s in self._shards):
            _collective(self._group, self._shards, lambda r, d: d.restore_layout())

    def shard_amps(self, shard: int) -> np.ndarray:
        self._identity_layout()
        return self._shards[shard].copy_amps()

    @property
    def amps(self) -> np.ndarray:
        if self._amps is None:
            self._identity_layout()
            a = np.concatenate([s.copy_amps() for s in self._shards])
            a.setflags(write=False)
            self._amps = a
        return self._amps

    def _copy_range(self, start: int, count: int) -> np.ndarray:
        self._identity_layout()
        L = 1 << self._shards[0].n_local
        parts = []
        while count > 0:
            s, off = divmod(start, L)
            take = min(count, L - off)
            parts.append(self._shards[s].copy_amps(off, take))
            start += take
            count -= take
        return np.concatenate(parts) if parts else np.empty(0, dtype=self._precision.dtype)

    def _reductions(self, weights: np.ndarray | None):
        if weights is not None and (self._cost is None or not np.array_equal(self._cost, weights)):
            w = np.asarray(weights, dtype=np.float64)
            _collective(self._group, self._shards, lambda r, d: (d.set_cost(w), d.recompute()))
            self._cost = np.array(w)
        return _collective(self._group, self._shards, lambda r, d: d.reduce())[0]

    def _draw(self, u: np.ndarray) -> np.ndarray:
        return _collective(self._group, self._shards, lambda r, d: d.sample(u))[0]

    def _histogram(self, weights: np.ndarray, bins: int, lo: float, hi: float):
        w = np.asarray(weights, dtype=np.float64)

        def body(r, d):
            d.set_cost(w)
            d.set_histogram(bins, lo, hi)
            d.recompute()
            out = (d.histogram(), d.reduce())
            d.set_histogram(0)
            return out

        res = _collective(self._group, self._shards, body)
        self._cost = np.array(w)
        return res[0]

    def norm_squared(self) -> float:
        return float(self._reductions(None).sum_p)

    def norm_tolerance(self) -> float:
        eps = np.finfo(np.float32 if self._precision is Precision.FP32 else np.float64).eps
        return 10.0 * (1 << self.num_qubits) * float(eps)

    def probabilities(self) -> np.ndarray:
        a = self.amps.astype(np.complex128, copy=False)
        return (a.real ** 2 + a.imag ** 2).astype(np.float64)

    def save(self, path) -> None:
        """LQSV dump written by every shard's thread into its own byte range."""
        from .engine import lqsv_create, lqsv_write_range

        self._identity_layout()
        lqsv_create(path, self.num_qubits, self._precision)
        L = 1 << self._shards[0].n_local
        _collective(self._group, self._shards,
                    lambda r, d: lqsv_write_range(path, d, r * L, L, self._precision))

    def release(self) -> None:
        for s in self._shards:
            s.close(park=False)
        self._shards = []
        if self._group is not None:
            self._group.close()
            self._group = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.release()
        except Exception:
            pass


def _rows_from_timings(per_shard: list[tuple[list, str]], nq: int, G: int) -> list[GateTiming]:
    kinds = per_shard[0][1]
    g = G.bit_length() - 1
    rows = []
    for i, k in enumerate(kinds):
        ms = max(t[0][i] for t in per_shard) / 1e3
        if k in "TYW":
            rows.append(GateTiming(i, k, 0.0, ms, (G - 1) << (nq - g)))
        elif k == "X":
            rows.append(GateTiming(i, k, 0.0, ms, (1 << nq) if G > 1 else 0))
        else:
            rows.append(GateTiming(i, k, ms, 0.0, 0))
    return rows


def run_circuit_sharded(circuit: CircuitIR, plan: ShardPlan, precision: Precision | str = Precision.FP32,
                        memory_budget: int | None = None, devices: list[int] | None = None):
    """Run the circuit across plan.num_shards shard states; returns
    (state, TimingRecord) like the reference (sharded.py:299-385).

    devices: CUDA devices to place shards on (default: every visible one);
    shard s goes to devices[s * len(devices) // G], so neighbouring shards
    share a device and the rest talk over peer access.
    """
    precision = Precision.coerce(precision)
    if circuit.num_qubits != plan.nq:
        raise ValidationError(f"circuit has {circuit.num_qubits} qubits but plan covers {plan.nq}")
    check_memory(plan.nq, precision, memory_budget)
    layers = lower_circuit(circuit)
    p = int(layers.mixer.size)
    cost = getattr(circuit, "cost_weights", None)
    G = plan.num_shards
    wall0 = time.perf_counter()
    if not _engine_shards(plan.nq, G, precision, p):
        dev = _device_state(plan.nq, precision, memory_budget)
        if cost is not None:
            dev.set_cost(cost)
        dev.set_timing(True)
        dev.run(layers.phase, layers.mixer)
        rows = _rows_from_timings([dev.timings()], plan.nq, 1)
        dev.set_timing(False)
        rec = TimingRecord(nq=plan.nq, p=circuit.p, num_shards=G, wall_seconds=time.perf_counter() - wall0,
                           gates=rows)
        return StateVector._wrap(plan.nq, precision, dev, cost), rec
    if devices is None:
        devices = list(range(max(1, _native.device_count())))
    if not devices:
        raise ValidationError("no devices to place shards on")
    group = _native.ShardGroup(G)
    shards = []
    try:
        for s in range(G):
            d = _native.DeviceState.create_shard(plan.nq, precision.bytes_per_amplitude,
                                                 devices[s * len(devices) // G], s, group)
            shards.append(d)
            d.set_cost(cost if cost is not None else np.zeros(plan.nq * (plan.nq - 1) // 2))
            d.set_timing(True)
        _collective(group, shards, lambda r, d: d.run(layers.phase, layers.mixer))
        timings = [d.timings() for d in shards]
        for d in shards:
            d.set_timing(False)
    except BaseException:
        for d in shards:
            d.close(park=False)
        group.close()
        raise
    rows = _rows_from_timings(timings, plan.nq, G)
    rec = TimingRecord(nq=plan.nq, p=circuit.p, num_shards=G, wall_seconds=time.perf_counter() - wall0, gates=rows)
    return ShardedStateVector(plan, precision, group, shards, cost), rec


def load_statevector_sharded(path, plan: ShardPlan, devices: list[int] | None = None) -> ShardedStateVector:
    """An LQSV dump loaded into plan.num_shards shard states (one host thread
    per shard reads its own byte range), e.g. a dump larger than one device."""
    from .engine import lqsv_header, lqsv_read_range

    n, precision, _ = lqsv_header(path)
    if n != plan.nq:
        raise ValidationError(f"dump has {n} qubits but the plan covers {plan.nq}")
    G = plan.num_shards
    if devices is None:
        devices = list(range(max(1, _native.device_count())))
    group = _native.ShardGroup(G)
    shards = []
    try:
        for s in range(G):
            shards.append(_native.DeviceState.create_shard(n, precision.bytes_per_amplitude,
                                                           devices[s * len(devices) // G], s, group))
        L = 1 << shards[0].n_local
        zero = np.zeros(n * (n - 1) // 2)

        def body(r, d):
            lqsv_read_range(path, d, r * L, L, precision)
            d.set_cost(zero)
            d.recompute()

        _collective(group, shards, body)
    except BaseException:
        for d in shards:
            d.close(park=False)
        group.close()
        raise
    return ShardedStateVector(plan, precision, group, shards, None)


# ---------------------------------------------------------------------------
# scaling sweeps (sharded.py:388-450)


@dataclass
class SweepConfig:
    """Strong scaling (fixed nq, varying shard counts) or problem-size scaling
    (varying nq at fixed nq_local)."""

    mode: str = "strong"
    p: int = 3
    delta_beta: float = 0.2
    delta_gamma: float = 0.2
    seed: int = 1
    precision: Precision | str = Precision.FP32
    repeat: int = 1
    memory_budget: int | None = None
    nq: int | None = None
    shard_counts: tuple[int, ...] = (1, 2, 4)
    nq_values: tuple[int, ...] = ()
    nq_local: int | None = None

    def __post_init__(self) -> None:
        if self.mode not in ("strong", "size"):
            raise ValidationError(f"sweep mode must be 'strong' or 'size', got {self.mode!r}")
        if self.repeat < 1:
            raise ValidationError(f"repeat must be positive, got {self.repeat}")
        if self.mode == "strong" and (self.nq is None or not self.shard_counts):
            raise ValidationError("strong-scaling sweep needs nq and shard_counts")
        if self.mode == "size" and (not self.nq_values or self.nq_local is None):
            raise ValidationError("size sweep needs nq_values and nq_local")


def scaling_sweep(cfg: SweepConfig) -> list[TimingRecord]:
    params = LrQaoaParams(p=cfg.p, delta_beta=cfg.delta_beta, delta_gamma=cfg.delta_gamma)
    runs: list[tuple[CircuitIR, ShardPlan]] = []
    if cfg.mode == "strong":
        circ = build_circuit(generate_instance(cfg.nq, cfg.seed), params)
        runs = [(circ, plan_for_shard_count(cfg.nq, c)) for c in cfg.shard_counts]
    else:
        for nq in cfg.nq_values:
            if nq < cfg.nq_local:
                raise ValidationError(f"nq={nq} below nq_local={cfg.nq_local}")
            runs.append((build_circuit(generate_instance(nq, cfg.seed), params), plan_shards(nq, cfg.nq_local)))
    records = []
    for circ, plan in runs:
        for _ in range(cfg.repeat):
            sv, rec = run_circuit_sharded(circ, plan, cfg.precision, cfg.memory_budget)
            sv.release()
            records.append(rec)
    return records


__all__ = [
    "ExchangeStep", "GateTiming", "LAUNCH_KINDS", "ShardPlan", "ShardedStateVector", "SweepConfig",
    "TIMING_CSV_FIELDS", "TimingRecord", "exchange_steps", "exchange_volume", "plan_for_shard_count",
    "plan_shards", "remap_volume", "run_circuit_sharded", "scaling_sweep", "write_timing_csv",
    "load_statevector_sharded",
]
