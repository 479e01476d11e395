"""Small cases of every kernel family (n = 10-24, a few tiles each), checked
against the oracle.  compute-sanitizer is closed on the GPU pool, so these run
against the bounds-checked build instead (device asserts on tile indices,
global extents and the carved shared-memory layouts):

    python -m paper_2604_26423_b200.build --checked
    LRQ_LIB=paper_2604_26423_b200/_lib/liblrq_checked.so python scripts/sanitize_cases.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_26423_b200 as L  # noqa: E402
from oracle import lrq_oracle as O  # noqa: E402


def check(n, p, prec, dbeta=0.2):
    inst = L.solve_instance(L.generate_instance(n, 3))
    sv = L.run_circuit(L.build_circuit(L.generate_instance(n, 3), L.LrQaoaParams(p=p, delta_beta=dbeta)), prec)
    want = O.simulate(n, inst.weights(), p, "fp64", dbeta=dbeta)
    err = np.linalg.norm(sv.amps.astype(np.complex128) - want) / np.linalg.norm(want)
    assert err < (1e-10 if prec == "fp64" else 1e-5), (n, p, prec, err)
    L.exact_expected_r(sv, inst)
    L.sample(sv, 200, rng_seed=1)
    L.exact_cut_distribution(sv, inst, bins=64)
    sv.release()
    print("ok", n, p, prec, dbeta, err, flush=True)


# single CTA + classic / TMA / warp-decoupled sweeps, tiny whole-state kernel
for n, p, prec, db in [(10, 2, "fp64", 0.2), (14, 2, "fp32", 0.2), (15, 3, "fp64", 1.2), (16, 2, "fp32", 0.9),
                       (21, 2, "fp64", 0.2), (24, 2, "fp32", 0.2)]:
    check(n, p, prec, db)
# sharded: remap transports (fused, pipelined, serial) and the histogram
for mode in (("1", "1"), ("0", "1"), ("0", "0")):
    os.environ["LRQ_FUSED_REMAP"], os.environ["LRQ_PIPELINED_REMAP"] = mode
    circ = L.build_circuit(L.generate_instance(16, 4), L.LrQaoaParams(p=3, delta_beta=0.9))
    sv, _ = L.run_circuit_sharded(circ, L.plan_for_shard_count(16, 4), "fp64")
    inst = L.solve_instance(L.generate_instance(16, 4))
    L.exact_expected_r(sv, inst)
    L.sample(sv, 100, rng_seed=2)
    sv.release()
    print("ok sharded", mode, flush=True)
# gate-by-gate kernels, draw_indices, cut values
sv = L.zero_state(12, "fp64")
for q in range(12):
    L.apply_h(sv, q)
L.apply_rzz(sv, 0.3, 1, 7)
L.apply_rx(sv, 0.2, 5)
L.draw_indices(np.random.default_rng(0).random(5000), 100, L.derive_rng(0, "shots", 0))
inst = L.generate_instance(13, 1)
L.cut_values_range(inst, 0, 1 << 13)
print("ok misc", flush=True)
# the opt-in cluster-pair sweeps (complex64, n = 29: C8 + C8 groups)
os.environ["LRQ_CLUSTER"] = "1"
sv = L.run_circuit(L.build_circuit(L.generate_instance(29, 1), L.LrQaoaParams(p=2, delta_beta=0.9)), "fp32",
                   memory_budget=1 << 40)
print("ok cluster", sv.norm_squared(), flush=True)
sv.release()
os.environ["LRQ_CLUSTER"] = "0"
