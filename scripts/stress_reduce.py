"""Stress: the fused final-pass reductions must equal a separate read-only
recompute pass (same W, same state) on every run."""
import random
import sys
sys.path.insert(0, ".")
import paper_2604_26423_b200 as L
from paper_2604_26423_b200 import _native

random.seed(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
bad = 0
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 40):
    n = random.choice([13, 14, 17, 20, 23, 25, 26, 28])
    prec = random.choice(["fp32", "fp64"])
    p = random.choice([1, 2, 3, 4])
    db = random.choice([0.2, 1.1])
    inst = L.generate_instance(n, it)
    sv = L.run_circuit(L.build_circuit(inst, L.LrQaoaParams(p=p, delta_beta=db)), prec)
    r = sv.device_state.reduce()
    a = (r.sum_p, r.sum_p_cut, r.min_energy, r.argmax_cut)
    sv.device_state.recompute()
    q = sv.device_state.reduce()
    b = (q.sum_p, q.sum_p_cut, q.min_energy, q.argmax_cut)
    ok = abs(a[1] - b[1]) <= 1e-9 * abs(b[1]) and a[3] == b[3] and abs(a[0] - b[0]) < 1e-12
    if not ok:
        bad += 1
    print(it, n, prec, p, db, "OK" if ok else "MISMATCH", a, b, flush=True)
    if random.random() < 0.5:
        sv.release()
print("mismatches", bad)
