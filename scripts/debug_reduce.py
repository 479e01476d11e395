import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2604_26423_b200 as L
from paper_2604_26423_b200 import _native
n = int(sys.argv[1]); prec = sys.argv[2]
inst = L.generate_instance(n, 1)
circ = L.build_circuit(inst, L.LrQaoaParams(p=3))
lay = L.lower_circuit(circ)
pb = 8 if prec == "fp32" else 16
for trial in range(4):
    dev = _native.DeviceState(n, pb)
    dev.set_cost(inst.weights())
    dev.run(lay.phase, lay.mixer)
    r = dev.reduce()
    dev.recompute()
    q = dev.reduce()
    print(trial, "run:", r.sum_p, r.sum_p_cut, r.min_energy, r.argmax_cut, " recompute:", q.sum_p, q.sum_p_cut, q.min_energy, q.argmax_cut)
    dev.close(park=(trial % 2 == 1))
