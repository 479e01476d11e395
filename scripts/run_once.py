"""One engine run (for ncu captures): python scripts/run_once.py n p prec [LRQ env assignments]."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
for kv in sys.argv[4:]:
    k, v = kv.split("=", 1)
    os.environ[k] = v
import paper_2604_26423_b200 as L  # noqa: E402
from paper_2604_26423_b200 import _native  # noqa: E402

n, p, prec = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
inst = L.generate_instance(n, 1)
lay = L.lower_circuit(L.build_circuit(inst, L.LrQaoaParams(p=p)))
dev = _native.DeviceState(n, 8 if prec == "fp32" else 16)
dev.set_cost(inst.weights())
dev.run(lay.phase, lay.mixer)
print("sum_p", dev.reduce().sum_p)
