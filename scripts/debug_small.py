import sys
sys.path.insert(0, ".")
import paper_2604_26423_b200 as L
from paper_2604_26423_b200 import _native
for n, prec in ((14, "fp64"), (15, "fp32")):
    inst = L.generate_instance(n, 1)
    for trial in range(2):
        sv = L.run_circuit(L.build_circuit(inst, L.LrQaoaParams(p=3, delta_beta=0.3)), prec)
        r = sv.device_state.reduce()
        print(n, prec, trial, r.sum_p, r.sum_p_cut, r.min_energy, r.argmax_cut, flush=True)
        sv.release()
