"""Multi-GPU LR-QAOA: one process per GPU (torchrun), NCCL over NVLink.

Replaces the reference's thread-per-shard engine (lrqbench sharded.py:202-385)
for the hot path: rank r holds the 2^(n-g) amplitudes whose top g = log2(world)
bits equal r.  The cost phase is local on every rank; the mixer of the g
global qubits costs one NCCL all-to-all block transpose per layer
(DESIGN.md §5).  torch.distributed is only the bootstrap (it ships the NCCL
unique id); all device work is liblrq.so.

    torchrun --nproc-per-node 8 ... :
        dist.init_process_group("gloo")            # or "nccl"
        sv = run_circuit_distributed(circ, "fp64")  # collective
        r = sv.exact_expected_r(inst)               # collective
        shots = sv.sample(10_000, rng_seed=1)       # collective, same on all ranks
"""
from __future__ import annotations

import numpy as np

from . import _native
from .circuit import CircuitIR, lower_circuit
from .engine import Precision, ShotSet, check_memory
from .errors import StateError, ValidationError
from .problem import WmcInstance
from .rng import derive_rng


def _world(group):
    import torch.distributed as dist

    if not dist.is_initialized():
        raise StateError("run_circuit_distributed needs an initialised torch.distributed process group")
    return dist.get_rank(group), dist.get_world_size(group)


class DistStateVector:
    """This rank's shard of a distributed state (collective methods)."""

    def __init__(self, num_qubits, precision, dev, rank, world, group, cost):
        self.num_qubits = num_qubits
        self._precision = precision
        self._dev = dev
        self.rank = rank
        self.world = world
        self.n_local = num_qubits - (world.bit_length() - 1)
        self._group = group
        self._cost = cost

    @property
    def precision(self) -> Precision:
        return self._precision

    @property
    def device_state(self) -> _native.DeviceState:
        return self._dev

    def reduce(self):
        return self._dev.reduce()

    def norm_squared(self) -> float:
        return float(self.reduce().sum_p)

    def _reductions(self, weights: np.ndarray | None):
        """Collective: final-pass reductions for cost `weights` (None: the
        cost the run was fused with).  Another cost re-runs the read-only
        pass on every rank."""
        if weights is not None and (self._cost is None or not np.array_equal(self._cost, weights)):
            self._dev.set_cost(weights)
            self._dev.recompute()
            self._cost = np.array(weights, dtype=np.float64)
        return self._dev.reduce()

    def _draw(self, u: np.ndarray) -> np.ndarray:
        return self._dev.sample(u)

    def _histogram(self, weights: np.ndarray, bins: int, lo: float, hi: float):
        """Collective: one read-only pass with the E histogram on."""
        self._dev.set_cost(weights)
        self._dev.set_histogram(bins, lo, hi)
        try:
            self._dev.recompute()
            raw = self._dev.histogram()
            red = self._dev.reduce()
        finally:
            self._dev.set_histogram(0)
        self._cost = np.array(weights, dtype=np.float64)
        return raw, red

    def exact_expected_r(self, inst: WmcInstance) -> float:
        """Collective; same as engine.exact_expected_r(self, inst)."""
        if inst.num_vertices != self.num_qubits:
            raise ValidationError(
                f"instance has {inst.num_vertices} vertices, state has {self.num_qubits} qubits")
        if inst.optimal_cut is None:
            raise StateError("instance has no optimal cut; solve it first")
        return float(self._reductions(inst.weights()).sum_p_cut) / inst.optimal_cut.value

    def sample(self, n_shots: int, rng_seed: int) -> ShotSet:
        """Collective; the same global indices on every rank."""
        if n_shots < 1:
            raise ValidationError(f"shot count must be positive, got {n_shots}")
        u = derive_rng(rng_seed, "shots", 0).random(n_shots)
        return ShotSet(self.num_qubits, self._draw(u), int(rng_seed), "noiseless")

    def local_amps(self) -> np.ndarray:
        """This rank's shard (identity layout).  Collective when the run had
        an odd p: the final pass ran in the swapped layout and the remaining
        remap is made here (every rank must call it)."""
        self._dev.restore_layout()
        return self._dev.copy_amps()

    def gather_amps(self):
        """Full state on rank 0 (None elsewhere); small n only."""
        import torch
        import torch.distributed as dist

        local = torch.from_numpy(self.local_amps().view(np.float64 if self._precision is Precision.FP64
                                                        else np.float32).copy())
        parts = [torch.empty_like(local) for _ in range(self.world)] if self.rank == 0 else None
        dist.gather(local, parts, dst=0, group=self._group)
        if self.rank != 0:
            return None
        dt = np.complex128 if self._precision is Precision.FP64 else np.complex64
        return np.concatenate([p.numpy().view(dt) for p in parts])

    def save(self, path) -> None:
        """Collective LQSV dump (engine.py:279-293 format): rank 0 writes the
        header and sizes the file, then every rank streams its own shard into
        its byte range (ranks share the node's filesystem)."""
        import torch.distributed as dist

        from .engine import lqsv_create, lqsv_write_range

        self._dev.restore_layout()
        if self.rank == 0:
            lqsv_create(path, self.num_qubits, self._precision)
        dist.barrier(group=self._group)
        L = 1 << self.n_local
        lqsv_write_range(path, self._dev, self.rank * L, L, self._precision)
        dist.barrier(group=self._group)

    def release(self) -> None:
        """Park the shard for the next run_circuit_distributed of the same
        shape (all ranks release in step, so the pools stay symmetric)."""
        if self._dev is None:
            return
        key = (self.num_qubits, self._precision.bytes_per_amplitude, self._dev.device, self.rank, self.world,
               id(self._group))
        if key not in _DIST_POOL:
            _DIST_POOL[key] = self._dev
        else:
            self._dev.close()
        self._dev = None


# Parked shards: NCCL communicator setup costs far more than a small run, so
# a loop of run_circuit_distributed reuses one shard (and its communicator).
_DIST_POOL: dict = {}


def drain_dist_pool() -> None:
    while _DIST_POOL:
        _, dev = _DIST_POOL.popitem()
        dev.close()


REMAP_MODES = {0: "nccl", 1: "fused", 2: "peer"}


def enable_peer_remap(dev: _native.DeviceState, group=None) -> str:
    """Collective: exchange the ranks' buffer handles and map them
    (lrq_fused_setup).  Returns the remap transport every rank will use:
    "fused" (a spare buffer fits: the sweep before a remap stores straight
    into the owners' spares), "peer" (the state fills HBM: in-place pipelined
    block swaps over NVLink) or "nccl" (no peer mapping: pipelined
    send/recv)."""
    import torch.distributed as dist

    mine = dev.ipc_handles()
    world = dist.get_world_size(group)
    allh = [None] * world
    dist.all_gather_object(allh, mine, group=group)
    return REMAP_MODES[dev.fused_setup(b"".join(allh))]


def enable_fused_remap(dev: _native.DeviceState, group=None) -> bool:
    """Backward-compatible name: True when the fused form was enabled."""
    return enable_peer_remap(dev, group) == "fused"


def load_statevector_distributed(path, group=None, device: int | None = None) -> DistStateVector:
    """Collective: every rank reads its own shard of an LQSV dump straight
    into its device (no host holds the whole state)."""
    import torch.distributed as dist

    from .engine import lqsv_header, lqsv_read_range

    n, precision, _ = lqsv_header(path)
    rank, world = _world(group)
    if world & (world - 1):
        raise ValidationError(f"world size must be a power of two, got {world}")
    dev_index = _native.default_device() if device is None else int(device)
    if world == 1:
        dev = _native.DeviceState(n, precision.bytes_per_amplitude, dev_index)
    else:
        box = [_native.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0, group=group)
        dev = _native.DeviceState.create_dist(n, precision.bytes_per_amplitude, dev_index, rank, world, box[0])
        dev.remap_mode = enable_peer_remap(dev, group)
    L = 1 << (n - (world.bit_length() - 1))
    lqsv_read_range(path, dev, rank * L, L, precision)
    dev.set_cost(np.zeros(n * (n - 1) // 2))
    dev.recompute()
    return DistStateVector(n, precision, dev, rank, world, group, None)


def run_circuit_distributed(circuit: CircuitIR, precision: Precision | str = Precision.FP32, group=None,
                            device: int | None = None, memory_budget: int | None = None) -> DistStateVector:
    """Collective run of an LR-QAOA circuit over all ranks of `group`."""
    import torch.distributed as dist

    precision = Precision.coerce(precision)
    rank, world = _world(group)
    if world & (world - 1):
        raise ValidationError(f"world size must be a power of two, got {world}")
    n = circuit.num_qubits
    g = world.bit_length() - 1
    check_memory(n - g, precision, memory_budget)
    layers = lower_circuit(circuit)
    dev_index = _native.default_device() if device is None else int(device)
    dev = _DIST_POOL.pop((n, precision.bytes_per_amplitude, dev_index, rank, world, id(group)), None)
    if dev is None and world == 1:
        # one rank: the single-GPU engine (same methods, no communicator)
        dev = _native.DeviceState(n, precision.bytes_per_amplitude, dev_index, int(memory_budget or 0))
    if dev is None:
        box = [_native.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0, group=group)
        dev = _native.DeviceState.create_dist(n, precision.bytes_per_amplitude, dev_index, rank, world, box[0],
                                              int(memory_budget or 0))
        dev.remap_mode = enable_peer_remap(dev, group)
    cost = getattr(circuit, "cost_weights", None)
    dev.set_cost(cost if cost is not None else np.zeros(n * (n - 1) // 2))
    dev.set_search(getattr(circuit, "cost_optimum", None) is None)  # C* known: no max-cut search
    dev.run(layers.phase, layers.mixer)
    return DistStateVector(n, precision, dev, rank, world, group, cost)
