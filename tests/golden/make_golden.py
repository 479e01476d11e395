"""Generate the golden fixtures in this directory from the REAL reference.

This script imports the reference package from /root/reference/pkg/src, so it
only runs in the build container (the reference does not exist on GPU boxes).
Its outputs are small .npz files committed next to it; tests read only those.

Fixtures
--------
cfg1_n12.npz    config 1: generate_instance(12, 7), p=3, fp64 + fp32 final
                amplitudes, C*, x*, W, exact r, r_rand, sample(sv,1000,1),
                shot mean r, and the full cut_values diagonal (bit-exact pin).
small.npz       20 acceptance-#1 style cases (n=2..6, p=1..3, seed 100+case):
                final fp64 amplitudes, plus the triangle instance at p=3.
n14.npz         generate_instance(14, 5), p=4: fp64 + fp32 amplitudes, exact r.
n20.npz         generate_instance(20, 1), p=3, fp64: C*, x*, exact r,
                sample(sv, 10000, 1) indices, a strided amplitude subset.
rng.npz         first draws of the instance / shots streams for several seeds.
misc.json       gate counts, schedules, brute-force ties, cut tables.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import lrqbench as L  # noqa: E402
from lrqbench.problem import cut_values_range  # noqa: E402
from lrqbench.rng import derive_rng  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def _out(name):
    return os.path.join(HERE, name)


def cfg1():
    inst = L.solve_instance(L.generate_instance(12, 7))
    circ = L.build_circuit(inst, L.LrQaoaParams(p=3))
    sv64 = L.run_circuit(circ, "fp64")
    sv32 = L.run_circuit(circ, "fp32")
    shots = L.sample(sv64, 1000, rng_seed=1)
    shots32 = L.sample(sv32, 1000, rng_seed=1)
    z = np.arange(1 << 12, dtype=np.uint64)
    np.savez_compressed(
        _out("cfg1_n12.npz"),
        weights=np.array([w for _, _, w in inst.edges]),
        amps64=sv64.amps,
        amps32=sv32.amps,
        opt_bits=np.array(inst.optimal_cut.bitstring),
        opt_value=inst.optimal_cut.value,
        total_weight=inst.total_weight(),
        exact_r64=L.exact_expected_r(sv64, inst),
        exact_r32=L.exact_expected_r(sv32, inst),
        r_rand=L.random_baseline_expectation(inst),
        shots64=shots.indices,
        shots32=shots32.indices,
        mean_r64=L.approximation_ratio(inst, shots),
        cut_diag=L.cut_values(inst, z),
        cut_range=cut_values_range(inst, 0, 1 << 12),
    )


def small():
    out = {}
    for case in range(20):
        n = 2 + case % 5
        p = 1 + case % 3
        inst = L.generate_instance(n, seed=100 + case)
        circ = L.build_circuit(inst, L.LrQaoaParams(p=p))
        out[f"c{case}_amps"] = L.run_circuit(circ, "fp64").amps
        out[f"c{case}_amps32"] = L.run_circuit(circ, "fp32").amps
        out[f"c{case}_meta"] = np.array([n, p, 100 + case])
    tri = L.solve_instance(L.WmcInstance(3, ((0, 1, 0.5), (0, 2, 1.0), (1, 2, 0.25))))
    circ = L.build_circuit(tri, L.LrQaoaParams(p=3))
    sv = L.run_circuit(circ, "fp64")
    out["tri_amps"] = sv.amps
    out["tri_r"] = L.exact_expected_r(sv, tri)
    # non-default ramp amplitudes, including a large beta (tan(beta) > 1)
    inst = L.generate_instance(9, 77)
    circ = L.build_circuit(inst, L.LrQaoaParams(p=4, delta_beta=1.4, delta_gamma=0.9))
    out["bigbeta_amps"] = L.run_circuit(circ, "fp64").amps
    np.savez_compressed(_out("small.npz"), **out)


def n14():
    inst = L.solve_instance(L.generate_instance(14, 5))
    circ = L.build_circuit(inst, L.LrQaoaParams(p=4))
    sv64 = L.run_circuit(circ, "fp64")
    sv32 = L.run_circuit(circ, "fp32")
    np.savez_compressed(
        _out("n14.npz"),
        amps64=sv64.amps,
        amps32=sv32.amps,
        exact_r64=L.exact_expected_r(sv64, inst),
        exact_r32=L.exact_expected_r(sv32, inst),
        opt_value=inst.optimal_cut.value,
        opt_bits=np.array(inst.optimal_cut.bitstring),
    )


def n20():
    inst = L.solve_instance(L.generate_instance(20, 1), threads=8)
    circ = L.build_circuit(inst, L.LrQaoaParams(p=3))
    sv = L.run_circuit(circ, "fp64")
    shots = L.sample(sv, 10000, rng_seed=1)
    np.savez_compressed(
        _out("n20.npz"),
        opt_value=inst.optimal_cut.value,
        opt_bits=np.array(inst.optimal_cut.bitstring),
        exact_r=L.exact_expected_r(sv, inst),
        shots=shots.indices,
        mean_r=L.approximation_ratio(inst, shots),
        amp_stride=257,
        amps_strided=sv.amps[::257].copy(),
        norm_squared=sv.norm_squared(),
    )


def rng():
    out = {}
    for seed in (0, 1, 7, 12345, -3, 1 << 70):
        for n in (3, 12, 26):
            out[f"inst_{seed}_{n}"] = derive_rng(seed, "instance", n).random(8)
        out[f"shots_{seed}"] = derive_rng(seed, "shots", 0).random(8)
    np.savez_compressed(_out("rng.npz"), **{k.replace("-", "m"): v for k, v in out.items()})


def misc():
    tri = L.WmcInstance(3, ((0, 1, 0.5), (0, 2, 1.0), (1, 2, 0.25)))
    data = {
        "gate_counts": {f"{n},{p}": list(L.gate_counts(n, p)) for n, p in ((48, 3), (93, 3), (40, 3), (36, 3), (12, 3))},
        "schedule_p3": [list(L.build_schedule(L.LrQaoaParams(p=3)).betas),
                        list(L.build_schedule(L.LrQaoaParams(p=3)).gammas)],
        "triangle_cuts": {b: L.cut_value(tri, b) for b in ("000", "100", "010", "001", "110", "101", "011", "111")},
        "triangle_opt": list(L.optimal_cut_bruteforce(tri)),
        "tie_opt": list(L.optimal_cut_bruteforce(L.WmcInstance(2, ((0, 1, 0.3),)))),
        "bruteforce": {},
    }
    for n, seed in ((2, 0), (3, 1), (4, 2), (5, 3), (6, 4), (7, 5), (8, 6), (10, 9), (16, 4)):
        data["bruteforce"][f"{n},{seed}"] = list(L.optimal_cut_bruteforce(L.generate_instance(n, seed)))
    with open(_out("misc.json"), "w") as fh:
        json.dump(data, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    cfg1()
    small()
    n14()
    n20()
    rng()
    misc()
    print("golden fixtures written to", HERE)
