"""Golden noisy-trajectory results of the reference (noise.py), run in the
build container where the reference package is importable:

    noise.npz: for each case (n, p, eps, T, seed, precision):
      probs_<i>  noisy_expected_probs(...)           (channel average, float64)
      shots_<i>  run_noisy_ensemble(..., 50 shots)   (pooled indices)
      r_<i>      noisy_expected_r(...) for the solved instance
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from lrqbench import (DepolarizingConfig, LrQaoaParams, build_circuit, generate_instance,  # noqa: E402
                      noisy_expected_probs, noisy_expected_r, run_noisy_ensemble, solve_instance)

CASES = [(5, 2, 0.2, 3, 9, "fp64"), (6, 3, 0.05, 20, 4, "fp64"), (8, 3, 0.02, 40, 7, "fp32"),
         (10, 2, 0.3, 5, 11, "fp64"), (12, 3, 0.01, 8, 3, "fp32"), (6, 3, 0.0, 1, 5, "fp32")]

out = {}
for i, (n, p, eps, T, seed, prec) in enumerate(CASES):
    inst = solve_instance(generate_instance(n, seed))
    circ = build_circuit(inst, LrQaoaParams(p=p))
    cfg = DepolarizingConfig(eps, trajectories=T, rng_seed=seed)
    out[f"meta_{i}"] = np.array([n, p, T, seed], dtype=np.int64)
    out[f"eps_{i}"] = np.array(eps)
    out[f"prec_{i}"] = np.array(prec)
    out[f"probs_{i}"] = noisy_expected_probs(circ, cfg, prec)
    out[f"shots_{i}"] = run_noisy_ensemble(circ, cfg, 50, prec).indices
    out[f"r_{i}"] = np.array(noisy_expected_r(circ, inst, cfg, prec))
np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "noise.npz"), **out)
print("wrote noise.npz", len(CASES), "cases")
