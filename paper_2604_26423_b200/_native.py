"""ctypes binding of liblrq.so (include/lrq.h).

The engine has no CPU path: if the library is missing or no CUDA device is
visible, every compute entry point raises.  Return codes map onto the
reference's exception taxonomy (lrqbench errors.py:8-26): 2 -> ValidationError,
3 -> CapacityError, 4 -> StateError.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import AbortedRunError, CapacityError, StateError, ValidationError

_HERE = os.path.dirname(os.path.abspath(__file__))
# $LRQ_LIB selects another build of the same ABI (the bounds-checked
# _lib/liblrq_checked.so of `python -m paper_2604_26423_b200.build --checked`)
LIB_PATH = os.environ.get("LRQ_LIB") or os.path.join(_HERE, "_lib", "liblrq.so")
ABI_VERSION = 2

_lib = None
_lock = threading.Lock()

_c_int, _c_i64, _c_u64, _c_dbl = ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
_p = ctypes.c_void_p
_state_p = ctypes.c_void_p


class Reduction(ctypes.Structure):
    _fields_ = [("sum_p", ctypes.c_double), ("sum_p_cut", ctypes.c_double),
                ("min_energy", ctypes.c_double), ("argmax_cut", ctypes.c_uint64),
                ("max_energy", ctypes.c_double)]


_SIGNATURES = {
    "lrq_abi_version": ([], _c_int),
    "lrq_last_error": ([], ctypes.c_char_p),
    "lrq_device_count": ([ctypes.POINTER(_c_int)], _c_int),
    "lrq_describe_plan": ([_c_int, _c_int, _c_int, ctypes.c_char_p, ctypes.c_size_t], _c_int),
    "lrq_create": ([_c_int, _c_int, _c_int, _c_u64, ctypes.POINTER(_state_p)], _c_int),
    "lrq_destroy": ([_state_p], _c_int),
    "lrq_set_cost": ([_state_p, _p], _c_int),
    "lrq_run": ([_state_p, _c_int, _p, _p], _c_int),
    "lrq_run_fields": ([_state_p, _c_int, _p, _p, _p, _p], _c_int),
    "lrq_run_ex": ([_state_p, _c_int, _p, _p], _c_int),
    "lrq_permute_xor": ([_state_p, _c_u64], _c_int),
    "lrq_reset": ([_state_p, _c_int], _c_int),
    "lrq_apply_gate": ([_state_p, _c_int, _c_int, _c_int, _c_dbl], _c_int),
    "lrq_noisy_batch": ([_c_int, _c_int, _c_int, _c_int, _c_int, _p, _p, _p, _c_i64, _p, _p, _p], _c_int),
    "lrq_reduce": ([_state_p, ctypes.POINTER(Reduction)], _c_int),
    "lrq_recompute": ([_state_p], _c_int),
    "lrq_sample": ([_state_p, _p, _c_i64, _p], _c_int),
    "lrq_copy_amps": ([_state_p, _c_u64, _c_u64, _p], _c_int),
    "lrq_store_amps": ([_state_p, _c_u64, _c_u64, _p], _c_int),
    "lrq_cut_values": ([_c_int, _p, _p, _c_u64, _c_i64, _p, _c_int], _c_int),
    "lrq_max_cut": ([_c_int, _p, _c_int, ctypes.POINTER(_c_u64), ctypes.POINTER(_c_dbl)], _c_int),
    "lrq_cut_values_spin": ([_c_int, _p, _c_dbl, _c_u64, _c_i64, _p, _c_int], _c_int),
    "lrq_expected_cut": ([_c_int, _p, _c_dbl, _p, _c_u64, _p, _c_int], _c_int),
    "lrq_draw_indices": ([_p, _c_u64, _p, _c_i64, _p, _c_int], _c_int),
    "lrq_set_timing": ([_state_p, _c_int], _c_int),
    "lrq_set_histogram": ([_state_p, _c_int, _c_dbl, _c_dbl], _c_int),
    "lrq_set_search": ([_state_p, _c_int], _c_int),
    "lrq_get_histogram": ([_state_p, _p], _c_int),
    "lrq_get_timings": ([_state_p, _p, ctypes.c_char_p, _c_int, ctypes.POINTER(_c_int)], _c_int),
    "lrq_stream": ([_state_p, ctypes.POINTER(_p)], _c_int),
    "lrq_synchronize": ([_state_p], _c_int),
    "lrq_nccl_unique_id": ([_p, ctypes.c_size_t], _c_int),
    "lrq_create_dist": ([_c_int, _c_int, _c_int, _c_int, _c_int, _p, _c_u64, ctypes.POINTER(_state_p)], _c_int),
    "lrq_group_create": ([_c_int, ctypes.POINTER(_p)], _c_int),
    "lrq_group_destroy": ([_p], _c_int),
    "lrq_group_abort": ([_p], _c_int),
    "lrq_create_shard": ([_c_int, _c_int, _c_int, _c_int, _p, _c_u64, ctypes.POINTER(_state_p)], _c_int),
    "lrq_ipc_handles": ([_state_p, _p, ctypes.c_size_t], _c_int),
    "lrq_fused_setup": ([_state_p, _p, ctypes.POINTER(_c_int)], _c_int),
    "lrq_dist_info": ([_state_p, ctypes.POINTER(_c_int), ctypes.POINTER(_c_int), ctypes.POINTER(_c_int)], _c_int),
    "lrq_restore_layout": ([_state_p], _c_int),
    "lrq_dist_layout": ([_state_p, ctypes.POINTER(_c_int)], _c_int),
    "lrq_describe_dist_plan": ([_c_int, _c_int, _c_int, _c_int, ctypes.c_char_p, ctypes.c_size_t], _c_int),
    "lrq_dist_terms": ([_c_int, _c_int, _c_int, _c_int, _p, _p, _p, ctypes.POINTER(_c_dbl)], _c_int),
    "lrq_describe_remap": ([_c_int, _c_int, _c_int, ctypes.c_char_p, ctypes.c_size_t], _c_int),
    "lrq_describe_memory": ([_c_int, _c_int, _c_int, _c_int, ctypes.POINTER(_c_u64), ctypes.POINTER(_c_u64),
                             ctypes.POINTER(_c_u64)], _c_int),
}

IPC_HANDLE_BYTES = 256  # LRQ_IPC_HANDLE_BYTES

EXPORTED = tuple(_SIGNATURES)


def lib():
    """Load liblrq.so once; raise loudly if it has not been built."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build the CUDA engine with "
                    "`python -m paper_2604_26423_b200.build` (there is no CPU fallback)")
            h = ctypes.CDLL(LIB_PATH)
            for name, (args, res) in _SIGNATURES.items():
                fn = getattr(h, name)
                fn.argtypes = args
                fn.restype = res
            if h.lrq_abi_version() != ABI_VERSION:
                raise RuntimeError("liblrq.so ABI version mismatch; rebuild the engine")
            _lib = h
        return _lib


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = (lib().lrq_last_error() or b"").decode(errors="replace")
    if rc == 2:
        raise ValidationError(msg)
    if rc == 3:
        raise CapacityError(msg)
    if msg.startswith("aborted run"):  # a collective failed on this or another rank
        raise AbortedRunError(msg)
    raise StateError(msg)


def device_count() -> int:
    c = _c_int(0)
    rc = lib().lrq_device_count(ctypes.byref(c))
    return int(c.value) if rc == 0 else 0


def default_device() -> int:
    """Device for new states: $LRQ_DEVICE; else, under a torchrun launch
    (LOCAL_RANK set), the local rank modulo the visible devices, so one
    process per GPU lands on its own GPU; else 0."""
    if os.environ.get("LRQ_DEVICE"):
        return int(os.environ["LRQ_DEVICE"])
    lr = os.environ.get("LOCAL_RANK")
    if lr is not None and int(os.environ.get("LOCAL_WORLD_SIZE", os.environ.get("WORLD_SIZE", "1"))) > 1:
        n = device_count()
        return int(lr) % n if n > 0 else int(lr)
    return 0


def describe_plan(n: int, precision_bytes: int, p: int) -> str:
    buf = ctypes.create_string_buffer(1 << 20)
    check(lib().lrq_describe_plan(n, precision_bytes, p, buf, len(buf)))
    return buf.value.decode()


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def describe_dist_plan(n: int, log2_world: int, precision_bytes: int, p: int) -> str:
    buf = ctypes.create_string_buffer(1 << 20)
    check(lib().lrq_describe_dist_plan(n, log2_world, precision_bytes, p, buf, len(buf)))
    return buf.value.decode()


def dist_terms(n: int, log2_world: int, rank: int, perm: int, edges: np.ndarray):
    """A rank's local view (matrix, field, constant) of a lexicographic Z-Z
    coupling in permutation state perm (host-only; see lrq_dist.cuh)."""
    edges = np.ascontiguousarray(edges, dtype=np.float64)
    nl = n - log2_world
    m = np.empty((nl, nl))
    f = np.empty(nl)
    c = _c_dbl(0.0)
    check(lib().lrq_dist_terms(n, log2_world, rank, perm, ptr(edges), ptr(m), ptr(f), ctypes.byref(c)))
    return m, f, float(c.value)


def describe_remap(world: int, rank: int, mirror: int = -1) -> list:
    """The remap schedule of `rank` (host-only, lrq_describe_remap)."""
    import json

    buf = ctypes.create_string_buffer(1 << 16)
    check(lib().lrq_describe_remap(world, rank, mirror, buf, len(buf)))
    return json.loads(buf.value.decode())


def describe_memory(n: int, precision_bytes: int, world: int, p: int = 1) -> dict:
    """Device bytes one rank allocates (host-only accounting, lrq_describe_memory)."""
    a, b, c = _c_u64(0), _c_u64(0), _c_u64(0)
    check(lib().lrq_describe_memory(n, precision_bytes, world, p, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
    return {"state": int(a.value), "other": int(b.value), "spare": int(c.value)}


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check(lib().lrq_nccl_unique_id(buf, 128))
    return buf.raw


# One parked lrq_state per (n, precision, device): run_circuit in a loop then
# reuses the HBM allocation instead of cudaFree/cudaMalloc of the whole state.
# States of any size are parked (a 128 GiB n=33 state re-allocated every call
# costs as much as a third of the circuit); every native call that allocates
# device memory goes through _retry_capacity, which drains the pool and retries
# once when the allocation fails, so a parked state never blocks this library.
# Callers allocating HBM themselves call drain_pool() first.
_POOL: dict = {}
_POOL_MAX_BYTES = None


def drain_pool() -> None:
    """Free every parked device state."""
    while _POOL:
        _, h = _POOL.popitem()
        lib().lrq_destroy(h)


def _retry_capacity(rc_fn):
    """check(rc_fn()); on an out-of-memory error with states parked, drain
    the pool and call once more."""
    try:
        check(rc_fn())
    except CapacityError:
        if not _POOL:
            raise
        drain_pool()
        check(rc_fn())


class DeviceState:
    """Owning handle of one lrq_state (a state vector in HBM)."""

    def __init__(self, n: int, precision_bytes: int, device: int | None = None, budget: int = 0):
        self._h = None
        self.n = n
        self.precision_bytes = precision_bytes
        self.device = default_device() if device is None else int(device)
        self.n_local = n
        key = (n, precision_bytes, self.device)
        h = _POOL.pop(key, None)
        if h is not None:
            self._h = h
            self.set_cost(np.zeros(n * (n - 1) // 2))
            self.set_search(True)
            return
        h = _state_p()
        _retry_capacity(lambda: lib().lrq_create(n, precision_bytes, self.device, int(budget), ctypes.byref(h)))
        self._h = h

    @classmethod
    def create_dist(cls, n: int, precision_bytes: int, device: int, rank: int, world: int, nccl_id: bytes,
                    budget: int = 0) -> "DeviceState":
        """One rank's shard of a state distributed over `world` GPUs (collective:
        every rank calls this with the same nccl_id)."""
        self = cls.__new__(cls)
        self._h = None
        self.n = n
        self.precision_bytes = precision_bytes
        self.device = int(device)
        h = _state_p()
        idbuf = ctypes.create_string_buffer(nccl_id, 128)
        check(lib().lrq_create_dist(n, precision_bytes, self.device, rank, world, idbuf, int(budget),
                                    ctypes.byref(h)))  # collective: no local retry
        self._h = h
        self.n_local = n - (int(world).bit_length() - 1)
        self._dist = True
        return self

    @classmethod
    def create_shard(cls, n: int, precision_bytes: int, device: int, rank: int, group: "ShardGroup",
                     budget: int = 0) -> "DeviceState":
        """Shard `rank` of an in-process shard group (one host thread per shard)."""
        self = cls.__new__(cls)
        self._h = None
        self.n = n
        self.precision_bytes = precision_bytes
        self.device = int(device)
        h = _state_p()
        _retry_capacity(lambda: lib().lrq_create_shard(n, precision_bytes, self.device, rank, group.handle,
                                                       int(budget), ctypes.byref(h)))
        self._h = h
        self.n_local = n - (group.world.bit_length() - 1)
        self._dist = True
        return self

    def ipc_handles(self) -> bytes:
        buf = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
        check(lib().lrq_ipc_handles(self.handle, buf, IPC_HANDLE_BYTES))
        return buf.raw

    def fused_setup(self, all_handles: bytes) -> int:
        """Collective: map the peers' buffers; returns the remap transport
        (1 fused, 2 pipelined over peer memory, 0 NCCL send/recv)."""
        buf = ctypes.create_string_buffer(all_handles, len(all_handles))
        on = _c_int(0)
        check(lib().lrq_fused_setup(self.handle, buf, ctypes.byref(on)))
        return int(on.value)

    def close(self, park: bool = True) -> None:
        """Release the state (distributed shards are never parked)."""
        if getattr(self, "_dist", False):
            park = False
        self._close(park)

    @property
    def handle(self):
        if self._h is None:
            raise StateError("device state has been released")
        return self._h

    def _call(self, rc_fn) -> None:
        """check(rc_fn()), retried once after draining the pool on an
        out-of-memory error -- except for distributed / shard states, whose
        calls are collective (a retry on one rank would desynchronise them)."""
        if getattr(self, "_dist", False):
            check(rc_fn())
        else:
            _retry_capacity(rc_fn)

    def _close(self, park: bool = True) -> None:
        """Release the state; the allocation is parked for reuse unless the
        pool already holds one for this shape (or park=False)."""
        if self._h is not None and _lib is not None:
            key = (self.n, self.precision_bytes, self.device)
            if park and key not in _POOL and (_POOL_MAX_BYTES is None
                                              or (self.precision_bytes << self.n) <= _POOL_MAX_BYTES):
                _POOL[key] = self._h
            else:
                _lib.lrq_destroy(self._h)
        self._h = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    # -- engine calls ---------------------------------------------------------
    def set_cost(self, w: np.ndarray) -> None:
        w = np.ascontiguousarray(w, dtype=np.float64)
        check(lib().lrq_set_cost(self.handle, ptr(w)))

    def run(self, phase: np.ndarray, mixer: np.ndarray) -> None:
        phase = np.ascontiguousarray(phase, dtype=np.float64)
        mixer = np.ascontiguousarray(mixer, dtype=np.float64)
        self._call(lambda: lib().lrq_run(self.handle, int(mixer.size), ptr(phase), ptr(mixer)))

    def run_fields(self, phase: np.ndarray, field: np.ndarray, constant: np.ndarray, mixer: np.ndarray) -> None:
        """run() with per-layer single-Z fields (p x n) and constant phases (p)."""
        phase = np.ascontiguousarray(phase, dtype=np.float64)
        field = np.ascontiguousarray(field, dtype=np.float64)
        constant = np.ascontiguousarray(constant, dtype=np.float64)
        mixer = np.ascontiguousarray(mixer, dtype=np.float64)
        p = int(mixer.size)
        if field.size != p * self.n or constant.size != p:
            raise ValidationError(f"fields need shape ({p}, {self.n}) and constants ({p},)")
        self._call(lambda: lib().lrq_run_fields(self.handle, p, ptr(phase), ptr(field), ptr(constant), ptr(mixer)))

    def run_ex(self, phase: np.ndarray, mixer_q: np.ndarray) -> None:
        """run() with per-qubit mixer half-angles (p, n), equal up to sign per layer."""
        phase = np.ascontiguousarray(phase, dtype=np.float64)
        mixer_q = np.ascontiguousarray(mixer_q, dtype=np.float64)
        self._call(lambda: lib().lrq_run_ex(self.handle, int(mixer_q.shape[0]), ptr(phase), ptr(mixer_q)))

    def permute_xor(self, mask: int) -> None:
        check(lib().lrq_permute_xor(self.handle, int(mask)))

    def reset(self, which: int = 0) -> None:
        check(lib().lrq_reset(self.handle, int(which)))

    def apply_gate(self, kind: int, q0: int, q1: int = 0, theta: float = 0.0) -> None:
        check(lib().lrq_apply_gate(self.handle, int(kind), int(q0), int(q1), float(theta)))

    def reduce(self) -> Reduction:
        r = Reduction()
        self._call(lambda: lib().lrq_reduce(self.handle, ctypes.byref(r)))
        return r

    def recompute(self) -> None:
        check(lib().lrq_recompute(self.handle))

    def sample(self, u: np.ndarray) -> np.ndarray:
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.empty(u.size, dtype=np.uint64)
        self._call(lambda: lib().lrq_sample(self.handle, ptr(u), u.size, ptr(out)))
        return out

    def copy_amps(self, start: int = 0, count: int | None = None) -> np.ndarray:
        if count is None:
            count = (1 << self.n_local) - start
        dt = np.complex64 if self.precision_bytes == 8 else np.complex128
        out = np.empty(count, dtype=dt)
        check(lib().lrq_copy_amps(self.handle, start, count, ptr(out)))
        return out

    def store_amps(self, amps: np.ndarray, start: int = 0) -> None:
        dt = np.complex64 if self.precision_bytes == 8 else np.complex128
        amps = np.ascontiguousarray(amps, dtype=dt)
        check(lib().lrq_store_amps(self.handle, int(start), int(amps.size), ptr(amps)))

    def restore_layout(self) -> None:
        """Collective on a distributed / shard state: the identity layout back
        after an odd-p run (no-op otherwise)."""
        check(lib().lrq_restore_layout(self.handle))

    def layout(self) -> int:
        v = _c_int(0)
        check(lib().lrq_dist_layout(self.handle, ctypes.byref(v)))
        return int(v.value)

    def set_search(self, on: bool) -> None:
        """Whether reducing passes search the max cut (min E, argmin, max E)."""
        check(lib().lrq_set_search(self.handle, 1 if on else 0))

    def set_histogram(self, bins: int, lo: float = 0.0, hi: float = 1.0) -> None:
        """p-weighted E histogram of the next reducing pass (bins = 0: off)."""
        self._call(lambda: lib().lrq_set_histogram(self.handle, int(bins), float(lo), float(hi)))
        self.hist_bins = int(bins)

    def histogram(self) -> np.ndarray:
        """Raw fixed-point bins (units of 2^-60 probability; collective on ranks)."""
        out = np.zeros(max(1, getattr(self, "hist_bins", 0)), dtype=np.uint64)
        check(lib().lrq_get_histogram(self.handle, ptr(out)))
        return out

    def set_timing(self, on: bool) -> None:
        check(lib().lrq_set_timing(self.handle, 1 if on else 0))

    def timings(self):
        cnt = _c_int(0)
        check(lib().lrq_get_timings(self.handle, None, None, 0, ctypes.byref(cnt)))
        ms = np.zeros(max(1, cnt.value))
        kinds = ctypes.create_string_buffer(max(1, cnt.value) + 1)
        check(lib().lrq_get_timings(self.handle, ptr(ms), kinds, cnt.value, ctypes.byref(cnt)))
        return list(ms[: cnt.value]), kinds.raw[: cnt.value].decode()

    def stream(self) -> int:
        s = _p()
        check(lib().lrq_stream(self.handle, ctypes.byref(s)))
        return int(s.value or 0)

    def synchronize(self) -> None:
        check(lib().lrq_synchronize(self.handle))


class ShardGroup:
    """Owning handle of an lrq_group (in-process shard transport)."""

    def __init__(self, world: int):
        h = _p()
        check(lib().lrq_group_create(int(world), ctypes.byref(h)))
        self._h = h
        self.world = int(world)

    @property
    def handle(self):
        if self._h is None:
            raise StateError("shard group has been released")
        return self._h

    def abort(self) -> None:
        """Break the group: members blocked in a collective call return an error."""
        if self._h is not None:
            check(lib().lrq_group_abort(self._h))

    def close(self) -> None:
        if self._h is not None and _lib is not None:
            check(_lib.lrq_group_destroy(self._h))
        self._h = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass


def cut_values(n: int, w: np.ndarray, z: np.ndarray | None = None, start: int = 0, count: int = 0,
               device: int | None = None) -> np.ndarray:
    w = np.ascontiguousarray(w, dtype=np.float64)
    dev = default_device() if device is None else device
    if z is not None:
        z = np.ascontiguousarray(z, dtype=np.uint64)
        count = z.size
    out = np.empty(count, dtype=np.float64)
    if count:
        _retry_capacity(lambda: lib().lrq_cut_values(n, ptr(w), ptr(z) if z is not None else None, start, count,
                                                     ptr(out), dev))
    return out


def cut_values_spin(n: int, w: np.ndarray, half_total: float, start: int, count: int,
                    device: int | None = None) -> np.ndarray:
    """Spin-form cut values of [start, start+count) (lrq_cut_values_spin)."""
    w = np.ascontiguousarray(w, dtype=np.float64)
    dev = default_device() if device is None else device
    out = np.empty(int(count), dtype=np.float64)
    if count:
        _retry_capacity(lambda: lib().lrq_cut_values_spin(n, ptr(w), float(half_total), int(start), int(count),
                                                          ptr(out), dev))
    return out


def expected_cut_chunks(n: int, w: np.ndarray, half_total: float, probs: np.ndarray,
                        device: int | None = None) -> np.ndarray:
    """Per-2^16-chunk sums of p_z C(z) (lrq_expected_cut)."""
    w = np.ascontiguousarray(w, dtype=np.float64)
    probs = np.ascontiguousarray(probs, dtype=np.float64)
    dev = default_device() if device is None else device
    out = np.empty(max(1, probs.size >> 16), dtype=np.float64)
    _retry_capacity(lambda: lib().lrq_expected_cut(n, ptr(w), float(half_total), ptr(probs), probs.size, ptr(out),
                                                   dev))
    return out


def draw_indices(probs: np.ndarray, u: np.ndarray, device: int | None = None) -> np.ndarray:
    """Inverse-CDF draws over an explicit float64 distribution (lrq_draw_indices)."""
    probs = np.ascontiguousarray(probs, dtype=np.float64)
    u = np.ascontiguousarray(u, dtype=np.float64)
    dev = default_device() if device is None else device
    out = np.empty(u.size, dtype=np.uint64)
    _retry_capacity(lambda: lib().lrq_draw_indices(ptr(probs), probs.size, ptr(u), u.size, ptr(out), dev))
    return out


def max_cut(n: int, w: np.ndarray, device: int | None = None):
    w = np.ascontiguousarray(w, dtype=np.float64)
    dev = default_device() if device is None else device
    z = _c_u64(0)
    v = _c_dbl(0.0)
    _retry_capacity(lambda: lib().lrq_max_cut(n, ptr(w), dev, ctypes.byref(z), ctypes.byref(v)))
    return int(z.value), float(v.value)


def noisy_batch(n: int, precision_bytes: int, phase: np.ndarray, mixer: np.ndarray, xmask: np.ndarray,
                u: np.ndarray | None = None, want_probs: bool = True, device: int | None = None):
    """Batched small-n trajectories (lrq_noisy_batch): phase (T, p, E), mixer
    (T, p, n), xmask (T,), u (T, S) or None -> (probs (T, 2^n) | None,
    indices (T, S) | None)."""
    phase = np.ascontiguousarray(phase, dtype=np.float64)
    mixer = np.ascontiguousarray(mixer, dtype=np.float64)
    xmask = np.ascontiguousarray(xmask, dtype=np.uint32)
    T, p = mixer.shape[0], mixer.shape[1]
    dev = default_device() if device is None else int(device)
    probs = np.empty((T, 1 << n), dtype=np.float64) if want_probs else None
    shots = 0 if u is None else int(u.shape[1])
    idx = None
    if shots:
        u = np.ascontiguousarray(u, dtype=np.float64)
        idx = np.empty((T, shots), dtype=np.uint64)
    _retry_capacity(lambda: lib().lrq_noisy_batch(
        n, precision_bytes, dev, T, p, ptr(phase), ptr(mixer), ptr(xmask), shots, ptr(u) if shots else None,
        ptr(probs) if probs is not None else None, ptr(idx) if idx is not None else None))
    return probs, idx

