"""One engine run with the max-cut search off (the bench's timed final pass),
for ncu captures: python scripts/run_nosearch.py n p prec."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_26423_b200 as L  # noqa: E402
from paper_2604_26423_b200 import _native  # noqa: E402

n, p, prec = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
inst = L.generate_instance(n, 1)
lay = L.lower_circuit(L.build_circuit(inst, L.LrQaoaParams(p=p)))
dev = _native.DeviceState(n, 8 if prec == "fp32" else 16)
dev.set_cost(inst.weights())
dev.set_search(False)
dev.run(lay.phase, lay.mixer)
print("sum_p", dev.reduce().sum_p)
