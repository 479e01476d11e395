"""Generate config-2 (n=26, p=3, complex128) golden values from the REAL reference.

Run in the build container only (needs /root/reference); takes ~10 min single
threaded.  Output: tests/golden/cfg2_n26.npz (small: scalars, 1k shot indices,
and a strided 1/4096 subset of the final amplitudes).
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import lrqbench as L  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    n, seed, p = 26, 1, 3
    inst = L.generate_instance(n, seed)
    t0 = time.time()
    solved = L.solve_instance(inst, limit=26, threads=8)
    t_solve = time.time() - t0
    circ = L.build_circuit(solved, L.LrQaoaParams(p=p))
    t0 = time.time()
    sv = L.run_circuit(circ, "fp64", memory_budget=1 << 34)
    t_run = time.time() - t0
    r = L.exact_expected_r(sv, solved)
    shots = L.sample(sv, 1000, rng_seed=1)
    mean_r = L.approximation_ratio(solved, shots)
    stride = 4096
    np.savez_compressed(
        os.path.join(HERE, "cfg2_n26.npz"),
        n=n, seed=seed, p=p,
        opt_bits=np.array(solved.optimal_cut.bitstring),
        opt_value=solved.optimal_cut.value,
        total_weight=solved.total_weight(),
        exact_r=r,
        shots=shots.indices,
        mean_r=mean_r,
        amp_stride=stride,
        amps_strided=sv.amps[::stride].copy(),
        norm_squared=sv.norm_squared(),
        t_run_s=t_run, t_solve_s=t_solve,
    )
    print("n26 done", r, mean_r, solved.optimal_cut, t_run, t_solve)


if __name__ == "__main__":
    main()
