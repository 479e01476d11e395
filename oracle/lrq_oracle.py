"""numpy restatement of the reference LR-QAOA hot path (CPU ORACLE, tests only).

See ``oracle/__init__.py`` for who may import this module.  Every function
cites the reference file:line (``/root/reference/pkg/src/lrqbench/...``) whose
behaviour it restates.  The arithmetic is deliberately the same elementwise
numpy arithmetic as the reference (complex-scalar products on reshaped views,
sequential float64 cut accumulation, sequential ``cumsum`` CDF) so that the
oracle reproduces the reference bit for bit; the golden-vector tests pin that.
"""
from __future__ import annotations

import cmath
import math
import os
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

# --------------------------------------------------------------------------
# rng streams — rng.py:22-50

STREAM_CODES = {"instance": 0, "shots": 1, "trajectory": 2, "uniform": 3,
                "resample": 4, "classify": 5, "sweep": 6, "ideal": 7}


def stream(seed: int, name: str, *idx: int) -> np.random.Generator:
    """rng.py:43-45 — Philox keyed by SeedSequence(seed mod 2^64, (code, *idx))."""
    ss = np.random.SeedSequence(entropy=int(seed) % (1 << 64),
                                spawn_key=(STREAM_CODES[name],) + tuple(idx))
    return np.random.Generator(np.random.Philox(ss))


# --------------------------------------------------------------------------
# problem — problem.py:32-34, 90-101, 139-211, 242-264


def edge_pairs(n: int):
    """problem.py:32-34 — (i, j), i < j, lexicographic."""
    return [(a, b) for a in range(n) for b in range(a + 1, n)]


def instance_weights(n: int, seed: int) -> np.ndarray:
    """problem.py:90-101 — weights of generate_instance(n, seed), lex order."""
    return stream(seed, "instance", n).random(n * (n - 1) // 2)


def cut_diag(n: int, w: np.ndarray, z) -> np.ndarray:
    """problem.py:139-149 — sequential float64 accumulation in edge order.

    acc_{k+1} = acc_k + w_k * bit, with w_k * bit exact (bit in {0, 1}).
    """
    z = np.asarray(z, dtype=np.uint64)
    acc = np.zeros(z.shape, dtype=np.float64)
    for (a, b), wk in zip(edge_pairs(n), w):
        crossing = ((z >> np.uint64(a)) ^ (z >> np.uint64(b))) & np.uint64(1)
        acc += float(wk) * crossing
    return acc


def weight_matrix(n: int, w: np.ndarray) -> np.ndarray:
    m = np.zeros((n, n))
    for (a, b), wk in zip(edge_pairs(n), w):
        m[a, b] = m[b, a] = wk
    return m


def cut_block(n: int, w: np.ndarray, lo: int, hi: int) -> np.ndarray:
    """problem.py:158-171 — spin form W/2 - s^T A s / 4 on [lo, hi)."""
    a = weight_matrix(n, w)
    half = 0.5 * float(sum(float(x) for x in w))
    z = np.arange(lo, hi, dtype=np.uint64)
    bits = ((z[:, None] >> np.arange(n, dtype=np.uint64)[None, :]) & np.uint64(1))
    s = 1.0 - 2.0 * bits.astype(np.float64)
    return half - 0.25 * np.einsum("ij,ij->i", s @ a, s)


def brute_force(n: int, w: np.ndarray, chunk_bits: int = 16):
    """problem.py:174-211 — argmax over all z (ties -> lowest index), then the
    value re-evaluated with the sequential form.  Returns (index, value)."""
    total = 1 << n
    step = 1 << min(chunk_bits, n)
    best_v, best_z = None, None
    for lo in range(0, total, step):
        v = cut_block(n, w, lo, min(lo + step, total))
        k = int(np.argmax(v))
        if best_v is None or v[k] > best_v or (v[k] == best_v and lo + k < best_z):
            best_v, best_z = float(v[k]), lo + k
    return best_z, float(cut_diag(n, w, [best_z])[0])


def bits_of(z: int, n: int) -> str:
    """problem.py:119-120 — vertex 0 leftmost."""
    return "".join("1" if (z >> k) & 1 else "0" for k in range(n))


# --------------------------------------------------------------------------
# schedule — circuit.py:58-63, 105-122


def ramp(p: int, dbeta: float = 0.2, dgamma: float = 0.2):
    """circuit.py:58-63."""
    betas = [(1.0 - k / p) * dbeta for k in range(p)]
    gammas = [((k + 1) / p) * dgamma for k in range(p)]
    return betas, gammas


def gate_list(n: int, w: np.ndarray, p: int, dbeta: float = 0.2, dgamma: float = 0.2):
    """circuit.py:105-122 — ("H", q) / ("RZZ", i, j, theta) / ("RX", q, theta)."""
    betas, gammas = ramp(p, dbeta, dgamma)
    ops = [("H", q) for q in range(n)]
    for beta, gamma in zip(betas, gammas):
        for (a, b), wk in zip(edge_pairs(n), w):
            ops.append(("RZZ", a, b, 2.0 * gamma * float(wk)))
        for q in range(n):
            ops.append(("RX", q, -2.0 * beta))
    return ops


# --------------------------------------------------------------------------
# dense per-gate engine — engine.py:99-110, 128-166, 198-207


class DenseOracle:
    """Flat 2^n array, qubit k at bit k; kernels act in place on views.

    ``threads > 1`` partitions each gate's view along an axis across a thread
    pool (numpy ufuncs release the GIL); each element receives exactly the same
    operation as in the single-threaded reference, so results are identical.
    """

    def __init__(self, n: int, precision: str = "fp64", threads: int = 1):
        self.n = n
        self.dtype = np.dtype(np.complex128 if precision == "fp64" else np.complex64)
        self.amps = np.zeros(1 << n, dtype=self.dtype)
        self.amps[0] = 1.0
        self.threads = max(1, int(threads))
        self._pool = ThreadPoolExecutor(self.threads) if self.threads > 1 else None

    def close(self):
        if self._pool is not None:
            self._pool.shutdown()
            self._pool = None

    # -- partitioned execution helpers --------------------------------------
    def _split(self, view: np.ndarray, fn):
        """Run fn(subview) over chunks of the longest of the first/last axis."""
        if self._pool is None:
            fn(view)
            return
        axis = 0 if view.shape[0] >= view.shape[-1] else view.ndim - 1
        size = view.shape[axis]
        parts = min(self.threads, size)
        bounds = [size * k // parts for k in range(parts + 1)]
        futs = []
        for lo, hi in zip(bounds[:-1], bounds[1:]):
            sl = [slice(None)] * view.ndim
            sl[axis] = slice(lo, hi)
            futs.append(self._pool.submit(fn, view[tuple(sl)]))
        for f in futs:
            f.result()

    # -- kernels -------------------------------------------------------------
    def h(self, q: int):
        """engine.py:128-134."""
        r = self.dtype.type(1.0 / math.sqrt(2.0))

        def body(v):
            lo = v[:, 0, :].copy()
            hi = v[:, 1, :]
            v[:, 0, :] = (lo + hi) * r
            v[:, 1, :] = (lo - hi) * r

        self._split(self.amps.reshape(-1, 2, 1 << q), body)

    def rx(self, q: int, theta: float):
        """engine.py:137-144 — [[c, s], [s, c]], c=cos(t/2), s=-i sin(t/2)."""
        c = self.dtype.type(math.cos(theta / 2.0))
        s = self.dtype.type(-1j * math.sin(theta / 2.0))

        def body(v):
            lo = v[:, 0, :].copy()
            hi = v[:, 1, :]
            v[:, 0, :] = c * lo + s * hi
            v[:, 1, :] = s * lo + c * hi

        self._split(self.amps.reshape(-1, 2, 1 << q), body)

    def rzz(self, qa: int, qb: int, theta: float):
        """engine.py:147-155 — equal bits e^{-i t/2}, differing e^{+i t/2}."""
        lo_q, hi_q = min(qa, qb), max(qa, qb)
        same = self.dtype.type(cmath.exp(-0.5j * theta))
        diff = self.dtype.type(cmath.exp(0.5j * theta))

        def body(v):
            v[:, 0, :, 0, :] *= same
            v[:, 1, :, 1, :] *= same
            v[:, 0, :, 1, :] *= diff
            v[:, 1, :, 0, :] *= diff

        self._split(self.amps.reshape(-1, 2, 1 << (hi_q - lo_q - 1), 2, 1 << lo_q), body)

    def apply(self, op):
        if op[0] == "H":
            self.h(op[1])
        elif op[0] == "RX":
            self.rx(op[1], op[2])
        else:
            self.rzz(op[1], op[2], op[3])

    def run(self, ops):
        for op in ops:
            self.apply(op)
        return self.amps

    # -- observables ---------------------------------------------------------
    def probabilities(self) -> np.ndarray:
        """engine.py:94-96 — float64 |a|^2."""
        a = self.amps.astype(np.complex128, copy=False)
        return (a.real ** 2 + a.imag ** 2).astype(np.float64)


def simulate(n: int, w: np.ndarray, p: int, precision: str = "fp64",
             dbeta: float = 0.2, dgamma: float = 0.2, threads: int = 1) -> np.ndarray:
    """engine.py:198-207 — run_circuit(build_circuit(inst, params))."""
    eng = DenseOracle(n, precision, threads)
    try:
        return eng.run(gate_list(n, w, p, dbeta, dgamma))
    finally:
        eng.close()


def probabilities(amps: np.ndarray) -> np.ndarray:
    """engine.py:94-96."""
    a = amps.astype(np.complex128, copy=False)
    return (a.real ** 2 + a.imag ** 2).astype(np.float64)


def expected_cut(n: int, w: np.ndarray, probs: np.ndarray, chunk: int = 1 << 16) -> float:
    """engine.py:214-226 without the final division: sum_z p_z C(z) per chunk."""
    total = 0.0
    for lo in range(0, probs.size, chunk):
        hi = min(lo + chunk, probs.size)
        total += float(probs[lo:hi] @ cut_block(n, w, lo, hi))
    return total


def draw(probs: np.ndarray, u: np.ndarray) -> np.ndarray:
    """engine.py:254-263 — sequential cumsum, normalise by last, right search."""
    cdf = np.cumsum(probs)
    cdf /= cdf[-1]
    idx = np.searchsorted(cdf, u, side="right")
    return np.minimum(idx, cdf.size - 1).astype(np.uint64)


def shot_uniforms(rng_seed: int, shots: int) -> np.ndarray:
    """engine.py:272 — derive_rng(rng_seed, "shots", 0).random(shots)."""
    return stream(rng_seed, "shots", 0).random(shots)


def uniform_amplitude(n: int, precision: str) -> complex:
    """engine.py:99-110,128-134 — value of every amplitude after the H layer:
    n sequential products by fl(1/sqrt 2) in the state dtype."""
    dt = np.dtype(np.complex128 if precision == "fp64" else np.complex64)
    r = dt.type(1.0 / math.sqrt(2.0))
    v = dt.type(1.0)
    for _ in range(n):
        v = (v + dt.type(0.0)) * r
    return v


# --------------------------------------------------------------------------
# C restatement loader (oracle/cutdiag.c)

_LIB = None
_LIB_LOCK = threading.Lock()


def c_cut_diag(n: int, w: np.ndarray, z) -> np.ndarray:
    """Bit-exact sequential cut values via oracle/_build/liboracle_cut.so."""
    import ctypes

    global _LIB
    with _LIB_LOCK:
        if _LIB is None:
            path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_build", "liboracle_cut.so")
            _LIB = ctypes.CDLL(path)
            _LIB.oracle_cut_values.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                               ctypes.c_int64, ctypes.c_void_p]
    z = np.ascontiguousarray(z, dtype=np.uint64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    out = np.empty(z.shape, dtype=np.float64)
    _LIB.oracle_cut_values(n, w.ctypes.data, z.ctypes.data, z.size, out.ctypes.data)
    return out
