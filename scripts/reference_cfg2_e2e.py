"""BASELINE configs[1] end to end on the host with the reference package
itself (baseline/_ref lrqbench, unmodified) beside the same calls on the
GPU through this package: n=26, p=3, complex128, instance
generate_instance(26, 1), exact r and 1k samples.

    python scripts/reference_cfg2_e2e.py [--single]   -> one JSON line

The reference's C* comes from its own brute force (solve_instance,
limit 26, all host threads); the timed region is run_circuit(_sharded) ->
exact_expected_r -> sample, as a user of either package calls them.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(0, ROOT)

import lrqbench as R  # noqa: E402

import paper_2604_26423_b200 as L  # noqa: E402

n, p, seed, shots = 26, 3, 1, 1000
cores = len(os.sched_getaffinity(0))
G = 1
while G * 2 <= cores:
    G *= 2
out = {"workload": "BASELINE configs[1]: n=26 p=3 complex128, exact r + 1k samples", "host_cores": cores}

t0 = time.perf_counter()
inst = R.solve_instance(R.generate_instance(n, seed), limit=26, threads=cores)
out["reference_solve_s"] = time.perf_counter() - t0
circ = R.build_circuit(inst, R.LrQaoaParams(p=p))
budget = 1 << 40

t0 = time.perf_counter()
sv, rec = R.run_circuit_sharded(circ, R.plan_for_shard_count(n, G), "fp64", memory_budget=budget)
r_ref = R.exact_expected_r(sv, inst)
s_ref = R.sample(sv, shots, rng_seed=1)
out["reference_threaded"] = {"shards": G, "seconds": time.perf_counter() - t0, "exact_r": r_ref,
                             "sampled_r": R.approximation_ratio(inst, s_ref)}
del sv
if "--single" in sys.argv:
    t0 = time.perf_counter()
    sv = R.run_circuit(circ, "fp64", memory_budget=budget)
    r1 = R.exact_expected_r(sv, inst)
    R.sample(sv, shots, rng_seed=1)
    out["reference_single_thread"] = {"seconds": time.perf_counter() - t0, "exact_r": r1}
    del sv

# the same calls through this package on the GPU (the instance as the reference solved it)
linst = L.WmcInstance(n, inst.edges, inst.seed, L.OptimalCut(inst.optimal_cut.bitstring, inst.optimal_cut.value))
lcirc = L.build_circuit(linst, L.LrQaoaParams(p=p))
for _ in range(3):  # warm-up: library load, allocation
    lsv = L.run_circuit(lcirc, "fp64", memory_budget=budget)
    L.exact_expected_r(lsv, linst)
    L.sample(lsv, shots, rng_seed=1)
    del lsv
reps = 20
t0 = time.perf_counter()
for _ in range(reps):
    lsv = L.run_circuit(lcirc, "fp64", memory_budget=budget)
    r_gpu = L.exact_expected_r(lsv, linst)
    s_gpu = L.sample(lsv, shots, rng_seed=1)
    del lsv
t_gpu = (time.perf_counter() - t0) / reps
out["gpu"] = {"seconds": t_gpu, "exact_r": r_gpu, "sampled_r": L.approximation_ratio(linst, s_gpu),
              "identical_shots": int((s_gpu.indices == s_ref.indices).sum())}
out["r_rel_diff"] = abs(r_gpu - r_ref) / r_ref
out["speedup_vs_threaded_reference"] = out["reference_threaded"]["seconds"] / t_gpu
if "reference_single_thread" in out:
    out["speedup_vs_single_thread_reference"] = out["reference_single_thread"]["seconds"] / t_gpu
print(json.dumps(out), flush=True)
