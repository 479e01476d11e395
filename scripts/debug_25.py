import os, sys
sys.path.insert(0, ".")
import numpy as np
import paper_2604_26423_b200 as L
from paper_2604_26423_b200 import _native
n = 25
inst = L.generate_instance(n, 9)
circ = L.build_circuit(inst, L.LrQaoaParams(p=3, delta_beta=1.1))
c = L.cut_values_range(inst, 0, 1 << n)
for path in ("tma", "reg", "tma", "reg"):
    os.environ["LRQ_SWEEP_PATH"] = path
    sv = L.run_circuit(circ, "fp64")
    r = sv.device_state.reduce()
    a = sv.device_state.copy_amps()
    p = (a.real ** 2 + a.imag ** 2)
    truth = float(p @ c)
    sv.device_state.recompute()
    q = sv.device_state.reduce()
    print(path, "run", r.sum_p, r.sum_p_cut, r.min_energy, r.argmax_cut, "| recompute", q.sum_p_cut, "| host", p.sum(), truth, flush=True)
    sv.release()
