import os, sys
sys.path.insert(0, ".")
import numpy as np
import paper_2604_26423_b200 as L
from paper_2604_26423_b200 import _native

def tri():
    t = L.solve_instance(L.WmcInstance(3, ((0, 1, 0.5), (0, 2, 1.0), (1, 2, 0.25))))
    sv = L.run_circuit(L.build_circuit(t, L.LrQaoaParams(p=3)), "fp64"); sv.amps; L.exact_expected_r(sv, t)
    circ = L.build_circuit(L.generate_instance(9, 77), L.LrQaoaParams(p=4, delta_beta=1.4, delta_gamma=0.9))
    L.run_circuit(circ, "fp64").amps

def paths(n, prec, truth=False):
    inst = L.generate_instance(n, 9)
    circ = L.build_circuit(inst, L.LrQaoaParams(p=3, delta_beta=1.1))
    for path in ("tma", "reg"):
        os.environ["LRQ_SWEEP_PATH"] = path
        sv = L.run_circuit(circ, prec)
        r = sv.device_state.reduce()
        msg = f"{n} {prec} {path} run {r.sum_p:.15f} {r.sum_p_cut:.12f} {r.min_energy:.10f} {r.argmax_cut}"
        if truth:
            a = sv.device_state.copy_amps(); p = a.real.astype(np.float64) ** 2 + a.imag.astype(np.float64) ** 2
            c = L.cut_values_range(inst, 0, 1 << n)
            sv.device_state.recompute(); q = sv.device_state.reduce()
            msg += f" | recompute {q.sum_p_cut:.12f} host {float(p @ c):.12f}"
        print(msg, flush=True)
        sv.release()
    os.environ.pop("LRQ_SWEEP_PATH")

for rep in range(3):
    tri()
    paths(23, "fp32"); paths(26, "fp32"); paths(25, "fp64", truth=True)
