import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2604_26423_b200 as L
from paper_2604_26423_b200 import _native

def r28(tag):
    inst = L.generate_instance(28, 1)
    sv = L.run_circuit(L.build_circuit(inst, L.LrQaoaParams(p=3)), "fp64")
    red = sv.device_state.reduce()
    print(tag, red.sum_p, red.sum_p_cut, red.min_energy, red.argmax_cut, flush=True)
    sv.release()

r28("fresh-first")
tri = L.solve_instance(L.WmcInstance(3, ((0, 1, 0.5), (0, 2, 1.0), (1, 2, 0.25))))
sv = L.run_circuit(L.build_circuit(tri, L.LrQaoaParams(p=3)), "fp64")
print("tri r", L.exact_expected_r(sv, tri))
circ = L.build_circuit(L.generate_instance(9, 77), L.LrQaoaParams(p=4, delta_beta=1.4, delta_gamma=0.9))
sv2 = L.run_circuit(circ, "fp64"); a = sv2.amps
_native.drain_pool()
r28("after-small")
r28("again")
_native.drain_pool()
r28("after-drain")
