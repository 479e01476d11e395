"""Golden amplitudes of the reference's gate-by-gate engine on circuits that
are not LR-QAOA shaped (random H / RX / RZZ lists), run in the build
container where the reference package is importable -> gates.npz."""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from lrqbench import CircuitIR, GateOp, run_circuit  # noqa: E402

rng = np.random.default_rng(2024)
out = {}
for i, (n, m, prec) in enumerate([(5, 40, "fp64"), (8, 120, "fp64"), (11, 200, "fp32"), (11, 200, "fp64"),
                                  (14, 60, "fp64"), (14, 60, "fp32")]):
    kinds, qa, qb, th = [], [], [], []
    gates = []
    for _ in range(m):
        k = int(rng.integers(0, 3))
        a = int(rng.integers(0, n))
        b = int((a + 1 + rng.integers(0, n - 1)) % n)
        t = float(rng.uniform(-3.0, 3.0))
        if k == 0:
            gates.append(GateOp("H", (a,)))
        elif k == 1:
            gates.append(GateOp("RX", (a,), t))
        else:
            gates.append(GateOp("RZZ", (a, b), t))
        kinds.append(k)
        qa.append(a)
        qb.append(b)
        th.append(t)
    sv = run_circuit(CircuitIR(num_qubits=n, gates=gates), prec)
    out[f"n_{i}"] = np.array(n)
    out[f"prec_{i}"] = np.array(prec)
    out[f"gates_{i}"] = np.array([kinds, qa, qb], dtype=np.int64)
    out[f"theta_{i}"] = np.array(th)
    out[f"amps_{i}"] = sv.amps
np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "gates.npz"), **out)
print("wrote gates.npz")
